"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Bar (BASELINE.json north_star): unique/inverse/perm,
hit/miss/expire decisions, victims and counters bit-exact; rows within 1e-6
relative (fp32, per-key gradients summed in ascending batch position)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import Oracle, capacity, S_INF, LFU, LRU, LIGHT_LFU, PINNED  # noqa: E402
from workload import gen  # noqa: E402

LR = 0.01
RTOL = 1e-6


def _het():
    from paper_2112_07221_b200 import het
    return het


def assert_rows(a, b):
    np.testing.assert_allclose(a, b, rtol=RTOL, atol=1e-30)


class Pair:
    def __init__(self, R, D, frac, s, policy=LFU, persist=1, n_max=4096, track_div=1, pin=64):
        het = _het()
        self.R, self.D = R, D
        self.o = Oracle(R=R, D=D, C=capacity(frac, R), s=s, policy=policy, lfu_persist=persist,
                        track_div=track_div, pin_threshold=pin)
        self.g = het.HetCache(R, D, frac, s, policy, max_keys_per_call=n_max, lfu_persist=persist,
                              pin_threshold=pin)
        self.exact_rows = 0

    def step(self, t, keys, grads, check_logs=True, check_victims=True):
        kd = torch.from_numpy(keys).cuda()
        out = self.g.lookup(kd, t).cpu().numpy()
        oo = self.o.lookup(t, [keys])[0]
        assert_rows(out, oo)
        self.exact_rows += int((out == oo).all())
        if check_logs:
            gl = self.g.lookup_log()
            ol = self.o.lookup_log(0)
            n = keys.size
            assert np.array_equal(gl["unique"], ol["unique"])
            assert np.array_equal(gl["inverse"][:n], ol["inverse"])
            assert np.array_equal(gl["perm"][:n], ol["perm"])
            assert np.array_equal(gl["seg_off"], ol["seg_off"])
            assert np.array_equal(gl["status"], ol["status"]), (t, np.nonzero(gl["status"] != ol["status"]))
        if grads is not None:
            self.g.update(kd, torch.from_numpy(grads).cuda(), LR)
            self.o.update([grads], LR)
            if check_victims:
                gk, gd = self.g.victims()
                ok, od = self.o.victims(0)
                order = np.argsort(ok, kind="stable")
                assert np.array_equal(gk, ok[order]), t
                assert np.array_equal(gd, od[order]), t

    def compare_stats(self):
        gs = self.g.stats()
        os_ = self.o.stats(0)
        for k in ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses", "evictions", "dirty_pushes"]:
            assert gs[k] == os_[k], (k, gs[k], os_[k])
        assert gs["resident"] == self.o.cache_size(0)

    def compare_cache(self):
        gc = self.g.dump_cache()
        oc = self.o.dump_cache(0)
        assert np.array_equal(gc["keys"], oc["keys"])
        assert np.array_equal(gc["cs"], oc["cs"])
        assert np.array_equal(gc["cc"], oc["cc"])
        if self.g_policy == LIGHT_LFU:   # pinned entries carry the EP_PIN marker
            prim = np.where(oc["tick"] == PINNED, np.uint32(PINNED), oc["count"])
            assert self.g.stats()["pinned"] == int((oc["tick"] == PINNED).sum())
        else:
            prim = oc["count"] if self.g_policy == LFU else oc["tick"]
        assert np.array_equal(gc["prim"], prim)
        assert_rows(gc["v"], oc["v"])
        assert_rows(gc["p"], oc["p"])

    def finish(self):
        self.g.sync()
        self.o.flush()
        keys = np.arange(self.R, dtype=np.int64)
        gr, gcg = self.g.read_global(keys)
        orows, ocg = self.o.read_global(keys)
        assert np.array_equal(gcg, ocg)
        assert_rows(gr, orows)


def toy_keys(t, B=128, i=0):
    return gen.criteo_keys(i, t, 1, B, gen.cards_for("toy"))[0].numpy()


@pytest.mark.parametrize("policy,s,persist,frac", [
    (LFU, 10, 1, 0.1),       # BASELINE configs[0]
    (LRU, 10, 1, 0.1),
    (LFU, 0, 1, 0.1),
    (LFU, S_INF, 1, 0.1),
    (LFU, 3, 0, 0.05),
    (LRU, 100, 1, 0.3),
    (LFU, 10, 1, 0.0),       # no cache: HET Hybrid mode (R10)
])
@pytest.mark.parametrize("fused", [True, False])
def test_toy_full_parity(policy, s, persist, frac, fused, monkeypatch):
    """fused: the 3-kernel single-GPU step; unfused: the per-phase kernels
    (the multi-GPU / large-batch path)."""
    if not fused:
        monkeypatch.setenv("HET_NO_FUSED", "1")
    R, D, T = 1000, 8, 200
    p = Pair(R, D, frac, s, policy, persist)
    p.g_policy = policy
    for t in range(T):
        keys = toy_keys(t)
        grads = gen.grads(0, t, keys.size, D).numpy()
        p.step(t, keys, grads)
    p.compare_stats()
    p.compare_cache()
    p.finish()


@pytest.mark.parametrize("persist,pin,frac", [(1, 8, 0.1), (0, 3, 0.1), (1, 2, 0.05)])
@pytest.mark.parametrize("fused", [True, False])
def test_light_lfu_parity(persist, pin, frac, fused, monkeypatch):
    """Light-LFU (R27): promotions (ascending key, floor(C/2) cap --
    the cap binds with these thresholds), no count maintenance for pinned
    entries, pinned entries never victims; everything bit-exact vs the oracle."""
    if not fused:
        monkeypatch.setenv("HET_NO_FUSED", "1")
    R, D = 1000, 8
    p = Pair(R, D, frac, 10, LIGHT_LFU, persist, pin=pin)
    p.g_policy = LIGHT_LFU
    for t in range(150):
        keys = toy_keys(t)
        p.step(t, keys, gen.grads(0, t, keys.size, D).numpy())
        if t % 37 == 5:
            p.compare_cache()
    p.compare_stats()
    p.compare_cache()
    assert p.g.stats()["pinned"] == capacity(frac, R) // 2     # the cap binds
    p.finish()


@pytest.mark.parametrize("cb", ["0", "2"])
@pytest.mark.parametrize("fused", [True, False])
def test_lfu_generic_fallback(cb, fused, monkeypatch):
    """LFU with the count bitmaps disabled (0) or tiny (2): the exact generic
    selection runs instead of / after the bitmap path."""
    monkeypatch.setenv("HET_LFU_CB", cb)
    if not fused:
        monkeypatch.setenv("HET_NO_FUSED", "1")
    R, D = 1000, 8
    p = Pair(R, D, 0.1, 10, LFU, 1)
    p.g_policy = LFU
    for t in range(120):
        keys = toy_keys(t)
        p.step(t, keys, gen.grads(0, t, keys.size, D).numpy())
    p.compare_stats()
    p.compare_cache()
    p.finish()


def test_ragged_and_degenerate_calls():
    """n = 0, n = 1, all-duplicate batches, lookup without update, explicit Evict(k)."""
    R, D = 500, 12
    p = Pair(R, D, 0.02, 2, LFU)
    p.g_policy = LFU
    rng = np.random.default_rng(0)
    t = 0
    for n in [0, 1, 5, 3, 0, 64, 1]:
        keys = rng.integers(0, R, size=n).astype(np.int64)
        p.step(t, keys, gen.grads(0, t, n, D).numpy()); t += 1
    keys = np.full(40, 7, np.int64)
    p.step(t, keys, gen.grads(0, t, 40, D).numpy()); t += 1
    keys = rng.integers(0, 20, size=30).astype(np.int64)
    p.step(t, keys, None); t += 1                       # lookup only (no write)
    p.step(t, keys, gen.grads(0, t, 30, D).numpy()); t += 1
    ek = np.unique(keys)[:5]
    p.g.evict(torch.from_numpy(ek).cuda())
    p.o.evict_keys([ek])
    for _ in range(20):
        keys = rng.integers(0, R, size=rng.integers(0, 100)).astype(np.int64)
        p.step(t, keys, gen.grads(0, t, keys.size, D).numpy()); t += 1
    p.compare_stats()
    p.compare_cache()
    p.finish()


def test_dedup_paths_sizes():
    """The fused path's dedup kernels (multi-CTA rank count up to 8192, the
    cluster bitonic sort beyond) at sizes around their tile boundaries, with
    duplicates, keys 0 and R-1 and ragged tails: unique/inverse/perm/seg_off
    bit-exact vs the oracle."""
    R, D = 1 << 20, 4
    p = Pair(R, D, 0.01, 10, LFU, n_max=16384)
    p.g_policy = LFU
    rng = np.random.default_rng(7)
    sizes = [1, 2, 31, 32, 33, 1023, 4095, 4096, 4097, 8191, 8192, 8193, 12000, 16383, 16384]
    for t, n in enumerate(sizes):
        keys = rng.integers(0, R, size=n).astype(np.int64)
        keys[rng.integers(0, n, size=max(1, n // 4))] = keys[0]           # a heavy duplicate
        keys[rng.integers(0, n)] = 0
        keys[rng.integers(0, n)] = R - 1
        p.step(t, keys, gen.grads(0, t, n, D).numpy())
    p.compare_stats()
    p.finish()


def test_large_batch_multi_cta_dedup():
    """n > 16384 takes the multi-CTA sort/merge dedup path."""
    R, D = 50000, 4
    cards = gen.scaled_cards(R)
    p = Pair(R, D, 0.1, 5, LFU, n_max=40000)
    p.g_policy = LFU
    for t in range(6):
        keys = gen.criteo_keys(0, t, 1, 1500, cards)[0].numpy()   # n = 39000
        p.step(t, keys, gen.grads(0, t, keys.size, D).numpy())
    p.compare_stats()
    p.finish()


@pytest.mark.parametrize("D,B", [(128, 4096), (36, 2048), (8, 32768)])
def test_heavy_key_segment_reduce(D, B):
    """Per-phase path with Criteo-shaped batches large enough that small fields'
    keys occur thousands of times: keys with > 32 occurrences go through the
    TMA-ring heavy-key kernel (those with >= 2048 listed first), the rest through
    the half-warp kernel, concurrently.  Rows, clocks and pendings after every
    update must match the oracle's ordered sums.  B = 32768 (n = 851,968) is
    the largest batch of bench.py's hbm_sweep, at a small D."""
    R = 200000
    cards = gen.scaled_cards(R)
    n = B * 26
    p = Pair(R, D, 0.1, 4, LFU, n_max=n)
    p.g_policy = LFU
    counts = np.bincount(np.unique(gen.criteo_keys(0, 0, 1, B, cards)[0].numpy(), return_counts=True)[1])
    assert counts.size > 2048, "workload must contain keys with >= 2048 occurrences"
    for t in range(4):
        keys = gen.criteo_keys(0, t, 1, B, cards)[0].numpy()
        p.step(t, keys, gen.grads(0, t, keys.size, D).numpy())
    p.compare_stats()
    p.compare_cache()
    p.finish()


def test_heavy_key_wide_rows_unfused(monkeypatch):
    """16 KB rows (D=4096) on the per-phase path: one row per ring stage."""
    monkeypatch.setenv("HET_NO_FUSED", "1")
    R, D = 20000, 4096
    cards = gen.scaled_cards(R)
    p = Pair(R, D, 0.1, 100, LFU, n_max=4096, track_div=16)
    p.g_policy = LFU
    for t in range(6):
        keys = gen.criteo_keys(0, t, 1, 64, cards)[0].numpy()
        grads = gen.grads(0, t, keys.size, D).numpy()
        kd = torch.from_numpy(keys).cuda()
        out = p.g.lookup(kd, t).cpu().numpy()
        oo = p.o.lookup(t, [keys])[0]
        sel = _tracked_mask(keys, 16)
        assert_rows(out[sel], oo[sel])
        p.g.update(kd, torch.from_numpy(grads).cuda(), LR)
        p.o.update([grads], LR)
    p.compare_stats()
    keys = np.arange(R, dtype=np.int64)
    keys = keys[_tracked_mask(keys, 16)]
    p.g.sync(); p.o.flush()
    gr, gcg = p.g.read_global(keys)
    orows, ocg = p.o.read_global(keys)
    assert np.array_equal(gcg, ocg)
    assert_rows(gr, orows)


def test_eviction_slow_paths():
    """LRU ticks far above the initial base (slow threshold path) and a key
    bucket with more than 16384 tied candidates (slow sub-select path)."""
    R, D = 1 << 26, 4
    p = Pair(R, D, 100 / R, S_INF, LRU, n_max=24000)
    p.g_policy = LRU
    t0 = 10 ** 6
    keys = np.arange(0, 20000, dtype=np.int64)
    p.step(t0, keys, gen.grads(0, 0, keys.size, D).numpy())
    p.compare_stats()
    p2 = Pair(R, D, 100 / R, S_INF, LFU, n_max=24000)
    p2.g_policy = LFU
    p2.step(1, keys, gen.grads(0, 0, keys.size, D).numpy())
    p2.compare_stats()
    p2.compare_cache()


def test_errors_are_reported():
    het = _het()
    g = het.HetCache(100, 4, 0.1, 1, max_keys_per_call=64)
    k = torch.tensor([1, 2, 3], dtype=torch.int64, device="cuda")
    with pytest.raises(het.HetError) as e:
        g.update(k, torch.zeros(3, 4, device="cuda"), LR)       # write without read
    assert e.value.code == 3
    bad = torch.tensor([1, 100], dtype=torch.int64, device="cuda")
    g.lookup(bad, 0)
    with pytest.raises(het.HetError) as e:
        het.het_check(g.h)
    assert e.value.code == 2
    with pytest.raises(het.HetError):
        g.lookup(torch.zeros(65, dtype=torch.int64, device="cuda"), 1)  # n > n_max


def test_update_keys_must_be_the_lookups():
    """Alg. 3 writes the keys Alg. 2 read; a write of keys
    the read did not return is a protocol violation.
    Another length: HET_ERR_PROTOCOL at once.  The lookup's buffer, or a copy
    of its keys: accepted, results as the oracle's.  Other keys of the same
    length: sticky HET_ERR_PROTOCOL and the update is skipped -- no entry of
    the cache changes."""
    het = _het()
    R, D = 1000, 8
    o = Oracle(R=R, D=D, C=capacity(0.1, R), s=10)
    g = het.HetCache(R, D, 0.1, 10, max_keys_per_call=4096)
    for t in range(6):                       # the lookup's pointer / a device copy / a host copy
        keys = toy_keys(t)
        grads = gen.grads(0, t, keys.size, D).numpy()
        kd = torch.from_numpy(keys).cuda()
        assert_rows(g.lookup(kd, t).cpu().numpy(), o.lookup(t, [keys])[0])
        upd = [kd, kd.clone(), keys.copy()][t % 3]
        het.het_update(g.h, upd, keys.size, torch.from_numpy(grads).cuda(), LR)
        o.update([grads], LR)
        het.het_check(g.h)
    keys = toy_keys(6)
    kd = torch.from_numpy(keys).cuda()
    g.lookup(kd, 6)
    with pytest.raises(het.HetError) as e:   # another n
        g.update(kd[:-1], torch.zeros(keys.size - 1, D, device="cuda"), LR)
    assert e.value.code == 3
    before = g.dump_cache()
    other = kd.clone()
    other[keys.size // 2] = (other[keys.size // 2] + 1) % R
    if bool((other == kd).all()):
        other[0] = (other[0] + 1) % R
    g.update(other, torch.ones(keys.size, D, device="cuda"), LR)
    with pytest.raises(het.HetError) as e:
        het.het_check(g.h)
    assert e.value.code == 3
    after = g.dump_cache()
    for k in ["keys", "v", "p", "cs", "cc", "prim"]:
        assert np.array_equal(before[k], after[k]), k
    g.close()


def test_host_pointer_path():
    """Host buffers are staged by the library (the e2e path of bench.py)."""
    het = _het()
    R, D = 1000, 8
    o = Oracle(R=R, D=D, C=capacity(0.1, R), s=10)
    g = het.HetCache(R, D, 0.1, 10, max_keys_per_call=4096)
    for t in range(30):
        keys = toy_keys(t)
        grads = gen.grads(0, t, keys.size, D).numpy()
        out = np.zeros((keys.size, D), np.float32)
        het.het_lookup(g.h, keys, keys.size, t, out)
        torch.cuda.synchronize()
        assert_rows(out, o.lookup(t, [keys])[0])
        het.het_update(g.h, keys, keys.size, grads, LR)
        o.update([grads], LR)
    g.sync()


def test_host_pointer_path_update_beside_copy():
    """Host rows out, host gradients in, no synchronisation between the calls:
    the update runs on the library's stream beside the lookup's D2H of the
    rows (after the lookup's kernels) and the caller's stream waits for it.
    Rows, statistics and the flushed table equal the oracle's."""
    het = _het()
    R, D = 1000, 64
    o = Oracle(R=R, D=D, C=capacity(0.1, R), s=10)
    g = het.HetCache(R, D, 0.1, 10, max_keys_per_call=4096)
    for t in range(40):
        keys = torch.from_numpy(toy_keys(t)).pin_memory()
        grads = torch.from_numpy(gen.grads(0, t, keys.numel(), D).numpy()).pin_memory()
        out = torch.zeros((keys.numel(), D), dtype=torch.float32).pin_memory()
        het.het_lookup(g.h, keys, keys.numel(), t, out)
        het.het_update(g.h, keys, keys.numel(), grads, LR)
        torch.cuda.synchronize()
        assert_rows(out.numpy(), o.lookup(t, [keys.numpy()])[0])
        o.update([grads.numpy()], LR)
    gs, os_ = g.stats(), o.stats(0)
    for k in ["lookups", "keys", "unique", "hits", "exp1", "misses", "evictions", "dirty_pushes"]:
        assert gs[k] == os_[k], (k, gs[k], os_[k])
    g.sync()
    o.flush()
    rows = np.arange(R, dtype=np.int64)
    gr, gcg = g.read_global(rows)
    orows, ocg = o.read_global(rows)
    assert np.array_equal(gcg, ocg)
    np.testing.assert_allclose(gr, orows, rtol=1e-6, atol=1e-30)


@pytest.mark.parametrize("policy", [LFU, LRU])
def test_cuda_graph_replay_parity(policy):
    """A step captured into a CUDA graph (HET_CLOCK_AUTO: t = 0, 1, 2, ...)
    replays with the same results as the oracle."""
    het = _het()
    R, D = 1000, 8
    o = Oracle(R=R, D=D, C=capacity(0.1, R), s=10, policy=policy)
    g = het.HetCache(R, D, 0.1, 10, policy, max_keys_per_call=4096)
    n = 128 * 26
    kbuf = torch.empty(n, dtype=torch.int64, device="cuda")
    gbuf = torch.empty((n, D), dtype=torch.float32, device="cuda")
    out = torch.empty((n, D), dtype=torch.float32, device="cuda")
    t = 0
    for _ in range(5):                                   # eager steps
        keys = toy_keys(t)
        grads = gen.grads(0, t, n, D).numpy()
        kbuf.copy_(torch.from_numpy(keys)); gbuf.copy_(torch.from_numpy(grads))
        g.lookup(kbuf, het.HET_CLOCK_AUTO, out=out)
        g.update(kbuf, gbuf, LR)
        assert_rows(out.cpu().numpy(), o.lookup(t, [keys])[0])
        o.update([grads], LR)
        t += 1
    graph = g.capture_step(kbuf, gbuf, out, LR)
    for _ in range(40):                                  # replays
        keys = toy_keys(t)
        grads = gen.grads(0, t, n, D).numpy()
        kbuf.copy_(torch.from_numpy(keys)); gbuf.copy_(torch.from_numpy(grads))
        graph.replay()
        torch.cuda.synchronize()
        assert_rows(out.cpu().numpy(), o.lookup(t, [keys])[0])
        o.update([grads], LR)
        gk, _ = g.victims()
        assert np.array_equal(gk, np.sort(o.victims(0)[0]))
        t += 1
    p = Pair.__new__(Pair)
    p.g, p.o, p.R, p.D, p.g_policy = g, o, R, D, policy
    p.compare_stats()
    p.compare_cache()
    p.finish()


def test_wdl_full_size_graph_replay():
    """BASELINE configs[1] at full size (33,762,577 rows, D=128, cache 10 %,
    s=100, LFU, batch 128) in bench.py's launch configuration (CUDA-graph
    replay, HET_CLOCK_AUTO), from a cold cache through the first ~200
    eviction steps: statuses, victims, counters bit-exact every step; rows of
    a tracked 1/256 sample of keys (the oracle keeps rows only for them)."""
    het = _het()
    cards = gen.cards_for("criteo")
    R, D, B, frac, s = sum(cards), 128, 128, 0.1, 100
    n = B * 26
    C = capacity(frac, R)
    track = 256
    o = Oracle(R=R, D=D, C=C, s=s, track_div=track)
    g = het.HetCache(R, D, frac, s, LFU, max_keys_per_call=n)
    kbuf = torch.empty(n, dtype=torch.int64, device="cuda")
    gbuf = torch.empty((n, D), dtype=torch.float32, device="cuda")
    out = torch.empty((n, D), dtype=torch.float32, device="cuda")
    T = 6450
    chunk = 250
    graph = None
    evict_steps = 0
    for t0 in range(0, T, chunk):
        keys_blk = gen.criteo_keys(0, t0, chunk, B, cards).numpy()
        for j in range(chunk):
            t = t0 + j
            keys = keys_blk[j]
            grads = gen.grads(0, t, n, D)
            kbuf.copy_(torch.from_numpy(keys)); gbuf.copy_(grads)
            if graph is None:
                g.lookup(kbuf, het.HET_CLOCK_AUTO, out=out)
                g.update(kbuf, gbuf, LR)
                graph = g.capture_step(kbuf, gbuf, out, LR)
                # the eager step above already consumed t; the oracle follows
            else:
                graph.replay()
            oo = o.lookup(t, [keys])[0]
            o.update([grads.numpy()], LR)
            gl = g.lookup_log()
            ol = o.lookup_log(0)
            assert np.array_equal(gl["unique"], ol["unique"]), t
            assert np.array_equal(gl["status"], ol["status"]), t
            gk, gd = g.victims()
            ok, od = o.victims(0)
            order = np.argsort(ok, kind="stable")
            assert np.array_equal(gk, ok[order]) and np.array_equal(gd, od[order]), t
            evict_steps += ok.size > 0
            if j % 25 == 0:
                sel = _tracked_mask(keys, track)
                if sel.any():
                    np.testing.assert_allclose(out.cpu().numpy()[sel], oo[sel], rtol=RTOL, atol=1e-30)
    assert evict_steps > 100
    gs, os_ = g.stats(), o.stats(0)
    for k in ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses", "evictions", "dirty_pushes"]:
        assert gs[k] == os_[k], (k, gs[k], os_[k])


def _tracked_mask(keys, track):
    # the oracle's tracking rule: fmix(key ^ 0x7472616B) % track == 0
    M = (1 << 64) - 1
    out = np.zeros(len(keys), bool)
    for i, k in enumerate(keys.tolist()):
        x = (k ^ 0x7472616B) & M
        x ^= x >> 30; x = (x * 0xBF58476D1CE4E5B9) & M
        x ^= x >> 27; x = (x * 0x94D049BB133111EB) & M
        x ^= x >> 31
        out[i] = x % track == 0
    return out


@pytest.mark.parametrize("fused", [True, False])
def test_reddit_shaped_all_unique(fused, monkeypatch):
    """BASELINE configs[2] shape (GraphSAGE on Reddit): 232,965 node ids,
    14,208 distinct ids per worker-iteration (dedup on already-unique keys,
    P:687), D=128, cache 10 %, s=10 -- one worker; the fused lookup/update
    after the cluster dedup, and the per-phase kernels."""
    if not fused:
        monkeypatch.setenv("HET_NO_FUSED", "1")
    R, D, K = gen.REDDIT_ROWS, 128, 14208
    p = Pair(R, D, 0.1, 10, LFU, n_max=K, track_div=64)
    p.g_policy = LFU
    for t in range(12):
        keys = gen.reddit_keys(0, t, K).numpy()
        grads = gen.grads(0, t, K, D).numpy()
        kd = torch.from_numpy(keys).cuda()
        out = p.g.lookup(kd, t).cpu().numpy()
        oo = p.o.lookup(t, [keys])[0]
        sel = _tracked_mask(keys, 64)
        assert_rows(out[sel], oo[sel])
        gl, ol = p.g.lookup_log(), p.o.lookup_log(0)
        assert np.array_equal(gl["unique"], ol["unique"]) and np.array_equal(gl["status"], ol["status"])
        p.g.update(kd, torch.from_numpy(grads).cuda(), LR)
        p.o.update([grads], LR)
        gk, _ = p.g.victims()
        assert np.array_equal(gk, np.sort(p.o.victims(0)[0]))
    p.compare_stats()


@pytest.mark.parametrize("D,B,T", [(4096, 32, 8), (4096, 128, 16), (1024, 128, 24)])
def test_scale_shaped_wide_rows(D, B, T):
    """BASELINE configs[4] row shape (D=4096, 16 KB rows) on a scaled table:
    Criteo-shaped keys over 20,000 rows.  Wide rows run the decisions kernel
    (k_lookup_wide), the per-(position, slice) row moves (k_mv_as) and the
    per-thread cp.async segment reduce (k_seg_as) before the clock-only update;
    the flushed global table (c_g of every row, the tracked rows' values)
    equals the oracle's."""
    R = 20000
    cards = gen.scaled_cards(R)
    p = Pair(R, D, 0.1, 100, LFU, n_max=4096, track_div=16)
    p.g_policy = LFU
    for t in range(T):
        keys = gen.criteo_keys(0, t, 1, B, cards)[0].numpy()
        grads = gen.grads(0, t, keys.size, D).numpy()
        kd = torch.from_numpy(keys).cuda()
        out = p.g.lookup(kd, t).cpu().numpy()
        oo = p.o.lookup(t, [keys])[0]
        sel = _tracked_mask(keys, 16)
        assert_rows(out[sel], oo[sel])
        assert np.array_equal(p.g.lookup_log()["status"], p.o.lookup_log(0)["status"])
        p.g.update(kd, torch.from_numpy(grads).cuda(), LR)
        p.o.update([grads], LR)
    p.compare_stats()
    p.g.sync()
    p.o.flush()
    rows = np.arange(R, dtype=np.int64)
    gr, gcg = p.g.read_global(rows)
    orows, ocg = p.o.read_global(rows)
    assert np.array_equal(gcg, ocg)
    sel = _tracked_mask(rows, 16)
    assert_rows(gr[sel], orows[sel])


@pytest.mark.parametrize("B", [128, 400])   # n = 3,328 (multi-CTA rank dedup) and 10,400 (bucket dedup)
def test_prefetch_next_batch(B):
    """NEXT-1: het_prefetch runs the next lookup's dedup
    ahead -- here on a side stream while this step's update runs -- and the
    lookup with the same keys skips its own; every result stays the oracle's.
    A prefetch of other keys is ignored; host keys work; a key outside [0, R)
    found by the prefetch is reported by the lookup that consumes it."""
    het = _het()
    R, D, s, frac = 20000, 16, 3, 0.1
    cards = gen.scaled_cards(R)
    n = B * 26
    p = Pair(R, D, frac, s, LFU, n_max=n)
    p.g_policy = LFU
    side = torch.cuda.Stream()
    main = torch.cuda.current_stream()
    keys = [gen.criteo_keys(0, t, 1, B, cards)[0].numpy() for t in range(31)]
    kd = [torch.from_numpy(k).cuda() for k in keys]
    for t in range(30):
        out = p.g.lookup(kd[t], t).cpu().numpy()
        assert_rows(out, p.o.lookup(t, [keys[t]])[0])
        gl, ol = p.g.lookup_log(), p.o.lookup_log(0)
        assert np.array_equal(gl["unique"], ol["unique"]) and np.array_equal(gl["status"], ol["status"]), t
        assert np.array_equal(gl["inverse"][:n], ol["inverse"]), t
        side.wait_stream(main)
        with torch.cuda.stream(side):
            nxt = kd[t + 1] if t % 7 != 3 else kd[(t + 5) % 31]        # t % 7 == 3: a batch the next lookup is not
            het.het_prefetch(p.g.h, nxt, nxt.numel(), stream=side)
        grads = gen.grads(0, t, n, D).numpy()
        p.g.update(kd[t], torch.from_numpy(grads).cuda(), LR)
        p.o.update([grads], LR)
        main.wait_stream(side)
        gk, gd = p.g.victims()
        ok, od = p.o.victims(0)
        order = np.argsort(ok, kind="stable")
        assert np.array_equal(gk, ok[order]) and np.array_equal(gd, od[order]), t
    p.compare_stats()
    p.compare_cache()
    # host keys
    hk = keys[30]
    het.het_prefetch(p.g.h, hk, hk.size)
    out = np.zeros((hk.size, D), np.float32)
    het.het_lookup(p.g.h, hk, hk.size, 30, out)
    torch.cuda.synchronize()
    assert_rows(out, p.o.lookup(30, [hk])[0])
    p.finish()
    # a key outside [0, R) seen by the prefetch
    bad = kd[0].clone()
    bad[5] = R
    het.het_prefetch(p.g.h, bad, bad.numel())
    p.g.lookup(bad, 31)
    with pytest.raises(het.HetError) as e:
        het.het_check(p.g.h)
    assert e.value.code == 2
