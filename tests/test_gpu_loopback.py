"""N-worker parity on ONE GPU: the loopback group (include/het.h het_group_*)
runs N workers' state, kernels and peer-memory exchange records on device 0,
driven phase by phase (no NCCL, no spinning wait), against the N-worker CPU
oracle.  This is the driver-visible test of the multi-worker protocol:

- CheckValid condition (2) -- the owner's c_g against c_c + s, EXP2;
- the owner-side fused Evict(k)+Fetch(k) of expired hits and misses (R5);
- eviction pushes carried by the next round (U4 before the next L3, R1);
- explicit Cache.Evict(key) and the end-of-run flush over the exchange;
- Eq. 2, the dense mean, bitwise equal on every worker.

Bar (BASELINE.json north_star): unique keys, statuses, victims, counters and
clocks bit-exact; rows within 1e-6 relative."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.oracle import Oracle, capacity, LFU, LRU, LIGHT_LFU, S_INF  # noqa: E402
from workload import gen  # noqa: E402

LR = 0.01


def _het():
    from paper_2112_07221_b200 import het
    return het


def shape_cfg(shape):
    if shape == "reddit":      # BASELINE configs[2]: 14,208 distinct ids per worker (large-n dedup)
        return gen.REDDIT_ROWS, 128, 14208, None
    if shape == "wide":        # Criteo-shaped fields over 5,000 rows, 4 KB rows (D = 1024)
        return 5000, 1024, 4096, gen.scaled_cards(5000)
    if shape == "mixed":       # Criteo-shaped fields over 5,000 rows, relabelled per worker (below)
        return 5000, 8, 4096, gen.scaled_cards(5000)
    return 1000, 8, 4096, gen.cards_for("toy")   # BASELINE configs[0]


def batch_keys(shape, N, t, n_max, cards):
    if shape == "reddit":
        keys = [gen.reddit_keys(i, t, n_max).numpy() for i in range(N)]
    else:
        keys = [gen.criteo_keys(i, t, 1, 128, cards)[0].numpy() for i in range(N)]
    if shape == "mixed":                  # worker i relabels the rows by a bijection of its own, so a row hot
        mult = [1, 3, 7, 9]               # at one worker is cold at another: its c_g runs ahead of the cold
        keys = [(k * mult[i % 4] + 137 * i) % 5000 for i, k in enumerate(keys)]   # replicas -> EXP2
    if t % 7 == 3:                        # ragged: workers send different counts (worker 0 none at all)
        keys = [k[: (k.size // 33) * i] for i, k in enumerate(keys)]
    return keys


def run(N, shape="toy", policy=LFU, s=10, frac=0.1, T=40, pin=64, evict_at=(), check_cache=False):
    het = _het()
    R, D, n_max, cards = shape_cfg(shape)
    g = het.HetGroup(N, R, D, frac, s, policy, max_keys_per_call=n_max, pin_threshold=pin, dense_max=1 << 12)
    o = Oracle(R=R, D=D, C=capacity(frac, R), s=s, policy=policy, N=N, pin_threshold=pin)
    for t in range(T):
        keys = batch_keys(shape, N, t, n_max, cards)
        grads = [gen.grads(i, t, k.size, D).numpy() for i, k in enumerate(keys)]
        kd = [torch.from_numpy(k).cuda() for k in keys]
        outs = g.lookup(kd, t)
        oo = o.lookup(t, keys)
        for i in range(N):
            np.testing.assert_allclose(outs[i].cpu().numpy(), oo[i], rtol=1e-6, atol=1e-30, err_msg=f"t={t} i={i}")
            gl, ol = g.workers[i].lookup_log(), o.lookup_log(i)
            assert np.array_equal(gl["unique"], ol["unique"]), (t, i)
            assert np.array_equal(gl["inverse"][:keys[i].size], ol["inverse"]), (t, i)
            assert np.array_equal(gl["status"], ol["status"]), (t, i, np.nonzero(gl["status"] != ol["status"]))
        g.update(kd, [torch.from_numpy(x).cuda() for x in grads], LR)
        o.update(grads, LR)
        for i in range(N):
            gk, gd = g.workers[i].victims()
            ok, od = o.victims(i)
            order = np.argsort(ok, kind="stable")
            assert np.array_equal(gk, ok[order]), (t, i)
            assert np.array_equal(gd, od[order]), (t, i)
        if t in evict_at:                 # explicit Cache.Evict(key) of some keys of this batch
            ek = [np.unique(k)[::3].copy() for k in keys]
            g.evict([torch.from_numpy(x).cuda() for x in ek])
            o.evict_keys(ek)
        if check_cache and t % 13 == 12:
            compare_cache(g, o, N, policy)
    st = []
    for i in range(N):
        gs, os_ = g.workers[i].stats(), o.stats(i)
        for k in ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses", "evictions", "dirty_pushes"]:
            assert gs[k] == os_[k], (i, k, gs[k], os_[k])
        assert gs["resident"] == o.cache_size(i)
        assert gs["sticky_error"] == 0
        st.append(os_)
    g.sync()
    o.flush()
    for i in range(N):                    # the global table after the flush, shard by shard
        owned = np.arange(i, R, N, dtype=np.int64)
        gr, gcg = g.workers[i].read_global(owned)
        orows, ocg = o.read_global(owned)
        assert np.array_equal(gcg, ocg), i
        np.testing.assert_allclose(gr, orows, rtol=1e-6, atol=1e-30)
        assert g.workers[i].stats()["resident"] == 0
    return g, st


def compare_cache(g, o, N, policy):
    for i in range(N):
        gc, oc = g.workers[i].dump_cache(), o.dump_cache(i)
        assert np.array_equal(gc["keys"], oc["keys"]), i
        assert np.array_equal(gc["cs"], oc["cs"]), i
        assert np.array_equal(gc["cc"], oc["cc"]), i
        np.testing.assert_allclose(gc["v"], oc["v"], rtol=1e-6, atol=1e-30)
        np.testing.assert_allclose(gc["p"], oc["p"], rtol=1e-6, atol=1e-30)


def check_dense(g, N):
    """Eq. 2: buf_i <- mean_i(buf_i), identical bits on every worker; two
    epochs reuse each staging buffer; an odd count exercises the scalar tail."""
    for k, cnt in enumerate([1000, 1000, 998, 4096, 7]):
        xs = [torch.arange(cnt, device="cuda", dtype=torch.float32) * (i + 1) + k for i in range(N)]
        want = torch.zeros(cnt, dtype=torch.float32, device="cuda")
        for x in xs:                              # rank order, fp32, then * (1/N)
            want = want + x
        scale = torch.tensor(1.0) / torch.tensor(float(N))   # fl32(1/N), as the kernel's 1.0f / N
        want = want * scale.cuda()
        g.dense_allreduce(xs)
        torch.cuda.synchronize()
        for x in xs:
            assert torch.equal(x, want), (k, cnt)
    with pytest.raises(_het().HetError):          # beyond the staging (dense_max = 4096): no NCCL fallback here
        g.dense_allreduce([torch.zeros(8192, device="cuda") for _ in range(N)])


@pytest.mark.parametrize("N", [2, 3, 4])
@pytest.mark.parametrize("policy,s,frac", [(LFU, 10, 0.1), (LRU, 3, 0.05), (LFU, 0, 0.1), (LFU, S_INF, 0.2),
                                           (LFU, 1, 0.1)])
def test_loopback_parity(N, policy, s, frac):
    g, st = run(N, "toy", policy, s, frac, T=50, evict_at=(17,), check_cache=True)
    assert sum(x["dirty_pushes"] for x in st) > 0
    check_dense(g, N)
    g.close()


@pytest.mark.parametrize("N", [2, 3, 4])
@pytest.mark.parametrize("policy,s,frac", [(LFU, 1, 0.4), (LRU, 3, 0.3), (LFU, 2, 0.6)])
def test_loopback_exp2(N, policy, s, frac):
    """Workers with different hot rows: a replica validated by condition (1)
    is refused by condition (2) when its owner's c_g ran more than s ahead
     -- the EXP2 branch of the owner's check and of the requester's
    install, with the speculatively sent pending row applied (R5, R22)."""
    g, st = run(N, "mixed", policy, s, frac, T=60, evict_at=(23,), check_cache=True)
    assert sum(x["exp2"] for x in st) > 0
    g.close()


@pytest.mark.parametrize("N", [2, 4])
def test_loopback_unfused_path(N, monkeypatch):
    """HET_NO_FUSED: probe kernel + the non-fused exchange round (k_p2p_build /
    k_p2p_install) + gather + the per-phase eviction with k_p2p_pushes."""
    monkeypatch.setenv("HET_NO_FUSED", "1")
    g, st = run(N, "mixed", LFU, 2, 0.4, T=40, evict_at=(9,), check_cache=True)
    assert sum(x["exp2"] for x in st) > 0
    g.close()


@pytest.mark.parametrize("shape,N,policy,s,frac,T", [("reddit", 2, LFU, 10, 0.1, 8), ("reddit", 3, LFU, 1, 0.02, 6),
                                                     ("wide", 2, LFU, 3, 0.1, 20), ("wide", 3, LRU, 100, 0.05, 15),
                                                     ("toy", 3, LIGHT_LFU, 10, 0.1, 50)])
def test_loopback_shapes(shape, N, policy, s, frac, T):
    """BASELINE configs[2]-shaped batches (14,208 distinct ids per worker: the
    large-n dedup, thousands of misses and victims per round), 4 KB rows and
    light-LFU (R27)."""
    g, st = run(N, shape, policy, s, frac, T=T, pin=4)
    if policy == LIGHT_LFU:
        assert sum(g.workers[i].stats()["pinned"] for i in range(N)) == 0   # flushed: cache empty
    g.close()


def test_loopback_member_calls_are_rejected():
    """Collective calls on a loopback member must go through het_group_*."""
    het = _het()
    g = het.HetGroup(2, 1000, 8, 0.1, 10, max_keys_per_call=256)
    k = torch.arange(4, dtype=torch.int64, device="cuda")
    out = torch.empty((4, 8), device="cuda")
    with pytest.raises(het.HetError) as e:
        het.het_lookup(g.hs[0], k, 4, 0, out)
    assert e.value.code == 3
    with pytest.raises(het.HetError):
        het.het_group_lookup(g.hs[::-1], [k, k], [4, 4], 0, [out, out])   # not in rank order
    g.close()


def test_loopback_flush_rounds_split():
    """het_sync over the exchange when one key bin holds more dirty entries
    than a round carries (n_max = 32: 96 records per source): the bin is
    split again; the flushed table equals the oracle's (R16)."""
    het = _het()
    N, R, D, n, frac = 2, 400_000, 4, 32, 0.002
    g = het.HetGroup(N, R, D, frac, 5, LFU, max_keys_per_call=n)
    o = Oracle(R=R, D=D, C=capacity(frac, R), s=5, N=N)
    rng = np.random.default_rng(7)
    for t in range(60):
        keys = [rng.integers(0, 800, size=n).astype(np.int64) for _ in range(N)]
        grads = [gen.grads(i, t, n, D).numpy() for i in range(N)]
        kd = [torch.from_numpy(k).cuda() for k in keys]
        outs = g.lookup(kd, t)
        oo = o.lookup(t, keys)
        for i in range(N):
            np.testing.assert_allclose(outs[i].cpu().numpy(), oo[i], rtol=1e-6, atol=1e-30)
        g.update(kd, [torch.from_numpy(x).cuda() for x in grads], LR)
        o.update(grads, LR)
    assert min(o.cache_size(i) for i in range(N)) > 3 * n * 2   # more dirty rows in bin 0 than one round carries
    g.sync()
    o.flush()
    for i in range(N):
        owned = np.arange(i, 1000, N, dtype=np.int64)
        gr, gcg = g.workers[i].read_global(owned)
        orows, ocg = o.read_global(owned)
        assert np.array_equal(gcg, ocg), i
        np.testing.assert_allclose(gr, orows, rtol=1e-6, atol=1e-30)
    g.close()
