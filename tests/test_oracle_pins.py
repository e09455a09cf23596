"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU).

Every test here checks oracle/ against something other than itself: printed
worked examples (tests/golden/spec_examples.json, each cited), the paper's
closed rules, closed forms for a
single worker, conservation, and an independent
brute-force implementation (tests/brute.py, pin P14).
"""
import itertools
import math
import random

import numpy as np
import pytest

from oracle.oracle import Oracle, S_INF, LFU, LRU, LIGHT_LFU, PINNED, HIT, EXP1, EXP2, MISS, INIT_SEED
from brute import Brute, init_value

F32 = np.float32
LR = 0.01


def rnd_grads(rng, n, D):
    # exact small fp32 values (multiples of 2^-12 in [-1/8, 1/8))
    return (rng.integers(-512, 512, size=(n, D)).astype(np.float32) / F32(4096.0))


def zero_grads(keys_list, D):
    return [np.zeros((len(k), D), np.float32) for k in keys_list]


# ----------------------------------------------------------------------------- L1 dedup
def test_dedup_golden(golden):
    for ex in golden["dedup"]:
        o = Oracle(R=16, D=0, C=16, s=S_INF)
        o.lookup(0, [ex["keys"]])
        log = o.lookup_log(0)
        assert log["unique"].tolist() == ex["unique"], ex["cite"]
        assert np.diff(log["seg_off"]).tolist() == ex["multiplicity"], ex["cite"]
        # inverse maps every position to its key; perm groups positions by key, ascending
        keys = np.array(ex["keys"], np.int64)
        if keys.size:
            assert (log["unique"][log["inverse"]] == keys).all()
            assert (keys[log["perm"]] == np.repeat(log["unique"], np.diff(log["seg_off"]))).all()


def test_dedup_vs_textbook_unique():
    """P1: sorted unique / inverse equal numpy's unique; perm equals a stable argsort."""
    rng = np.random.default_rng(1)
    for n in [1, 2, 7, 100, 3328]:
        keys = rng.integers(0, max(2, n // 3), size=n)
        o = Oracle(R=n, D=0, C=n, s=S_INF)
        o.lookup(0, [keys])
        log = o.lookup_log(0)
        u, inv = np.unique(keys, return_inverse=True)
        assert (log["unique"] == u).all()
        assert (log["inverse"] == inv).all()
        assert (log["perm"] == np.argsort(keys, kind="stable")).all()
        assert log["seg_off"][0] == 0 and log["seg_off"][-1] == n


# ----------------------------------------------------------------------------- CheckValid
def _drive(o, t, per_worker_keys, update=True, D=0):
    o.lookup(t, per_worker_keys)
    if update:
        o.update(zero_grads(per_worker_keys, D) if D else None, LR)


def test_check_valid_vector_1(golden):
    """s=2, c_s=5, c_c=6, c_g=7 -> valid."""
    ex = golden["check_valid"][0]
    k = 3
    o = Oracle(R=8, D=0, C=8, s=2, N=2)
    t = 0
    # worker 1 alone: t0 miss (cs=cc=0), t1,t2 HIT, t3 EXP1 sync (cg=3, cs=cc=3), t4 HIT -> cc=5
    for _ in range(5):
        _drive(o, t, [[], [k]]); t += 1
    o.evict_keys([[], [k]])                                  # push cc=5 -> cg=5
    _drive(o, t, [[k], [k]]); t += 1                        # both fetch at cg=5, update -> cc=6
    _drive(o, t, [[], [k]]); t += 1                         # worker 1 HIT -> cc=7
    o.evict_keys([[], [k]])                                  # cg=7
    c = o.dump_cache(0)
    _, cg = o.read_global([k])
    assert (c["cs"][0], c["cc"][0], cg[0]) == (ex["cs"], ex["cc"], ex["cg"]), ex["cite"]
    o.lookup(t, [[k], []])
    assert o.lookup_log(0)["status"][0] == HIT, ex["cite"]


def test_check_valid_vector_2(golden):
    """s=0, c_s=5, c_c=6, c_g=6 -> invalid by condition 1 (EXP1)."""
    ex = golden["check_valid"][1]
    k = 5
    o = Oracle(R=8, D=0, C=8, s=0, N=2)
    t = 0
    for _ in range(5):                       # worker 1: every access syncs; ends cs=cc=4 -> cc=5
        _drive(o, t, [[], [k]]); t += 1
    o.evict_keys([[], [k]])                  # cg = 5
    _drive(o, t, [[k], [k]]); t += 1         # both: fetch cs=cc=5 -> cc=6
    o.evict_keys([[], [k]])                  # worker 1 pushes cc=6 -> cg=6
    c = o.dump_cache(0)
    _, cg = o.read_global([k])
    assert (c["cs"][0], c["cc"][0], cg[0]) == (ex["cs"], ex["cc"], ex["cg"]), ex["cite"]
    o.lookup(t, [[k], []])
    assert o.lookup_log(0)["status"][0] == EXP1, ex["cite"]


def test_check_valid_vector_3(golden):
    """s=1, c_s=5, c_c=5, c_g=7 -> invalid by condition 2 (EXP2).
    A clean resident entry (cc == cs) exists only after a lookup without update."""
    ex = golden["check_valid"][2]
    k = 6
    o = Oracle(R=8, D=0, C=8, s=1, N=2)
    t = 0
    # worker 1: t0 miss cs=cc=0 -> 1; t1 HIT -> 2; t2 EXP1 (2-0>1) sync cg=2 -> cs=cc=2 -> 3;
    # t3 HIT -> 4; t4 EXP1 sync cg=4 -> cs=cc=4 -> 5; evict -> cg=5
    for _ in range(5):
        _drive(o, t, [[], [k]]); t += 1
    o.evict_keys([[], [k]])
    _, cg = o.read_global([k]); assert cg[0] == 5
    _drive(o, t, [[k], []], update=False); t += 1       # worker 0 fetches, no write: cs=cc=5
    _drive(o, t, [[], [k]]); t += 1                     # worker 1 miss: cs=cc=5 -> 6
    _drive(o, t, [[], [k]]); t += 1                     # worker 1 HIT -> 7
    o.evict_keys([[], [k]])                             # cg = 7
    c = o.dump_cache(0)
    _, cg = o.read_global([k])
    assert (c["cs"][0], c["cc"][0], cg[0]) == (ex["cs"], ex["cc"], ex["cg"]), ex["cite"]
    o.lookup(t, [[k], []])
    assert o.lookup_log(0)["status"][0] == EXP2, ex["cite"]


# ----------------------------------------------------------------------------- Fetch / Evict clocks
@pytest.mark.parametrize("which", [0, 1])
def test_max_rule(golden, which):
    """S:133-134 / P:443: the server keeps c_g = max(c_g, c_c)."""
    ex = golden["max_rule"][which]
    k = 2
    o = Oracle(R=4, D=0, C=4, s=S_INF, N=2)
    t = 0
    for _ in range(ex["cg"]):
        _drive(o, t, [[k], [k]]); t += 1
    o.evict_keys([[], [k]])                  # worker 1 pushes cc = 4
    _, cg = o.read_global([k]); assert cg[0] == ex["cg"]
    # worker 0 was fetched at cg=0 and has cc = 4; reach cc = ex["cc"] (or push cc=3 from a fresh fetch)
    if ex["cc"] >= ex["cg"]:
        for _ in range(ex["cc"] - ex["cg"]):
            _drive(o, t, [[k], []]); t += 1
    else:
        o2 = Oracle(R=4, D=0, C=4, s=S_INF, N=2)
        t = 0
        for _ in range(ex["cc"]):
            _drive(o2, t, [[k], [k]]); t += 1
        for _ in range(ex["cg"] - ex["cc"]):
            _drive(o2, t, [[], [k]]); t += 1
        o2.evict_keys([[], [k]])             # cg = 4
        o = o2
    assert o.dump_cache(0)["cc"][0] == ex["cc"]
    o.evict_keys([[k], []])
    _, cg = o.read_global([k])
    assert cg[0] == ex["new_cg"], ex["cite"]


def test_fetch_sets_both_clocks(golden):
    """S:238 / P:439: a fetch sets c_s = c_c = c_g."""
    ex = golden["fetch_install"][0]
    k = 1
    o = Oracle(R=4, D=0, C=4, s=S_INF, N=2)
    for t in range(ex["cg"]):
        _drive(o, t, [[], [k]])
    o.evict_keys([[], [k]])
    o.lookup(100, [[k], []])                 # lookup only: the freshly fetched entry
    c = o.dump_cache(0)
    assert (c["cs"][0], c["cc"][0]) == (ex["cs"], ex["cc"]), ex["cite"]


# ----------------------------------------------------------------------------- Update / Clock
@pytest.mark.parametrize("idx", [0, 1])
def test_write_duplicates_sum_then_one_tick(golden, idx):
    """S:365 / S:259: duplicates' grads are summed (ascending position) before
    scaling by -lr, and the clock ticks once."""
    ex = golden["write_dup"][idx]
    D = 4
    k = 7
    o = Oracle(R=8, D=D, C=8, s=S_INF)
    keys = [k] * ex["occurrences"] + [3]
    out = o.lookup(0, [keys])[0]
    v0 = out[0].copy()
    g = np.array([[0.5, -0.25, 0.125, 1.0]] * len(keys), np.float32)
    g[-1] = 9.0
    o.update([g], LR)
    acc = F32(0.0)
    for _ in range(ex["occurrences"]):
        acc = F32(acc + g[0])
    expect = v0 + F32(F32(-LR) * acc)
    c = o.dump_cache(0)
    j = list(c["keys"]).index(k)
    assert (c["v"][j] == expect).all()
    assert c["cc"][j] - c["cs"][j] == ex["ticks"], ex["cite"]
    assert (c["p"][j] == F32(F32(-LR) * acc)).all()


# ----------------------------------------------------------------------------- Evict() policy
def test_evict_overflow_vectors(golden):
    """the LFU victim is the smallest count, LRU the oldest touch,
    ties go to the smaller key (R9)."""
    a, b, c, d = 10, 11, 12, 13
    # LFU {a:5, b:1, c:3}: all three resident at once, one over capacity 2 -> evict b
    ex = golden["evict_overflow"][0]
    o = Oracle(R=16, D=0, C=2, s=S_INF, policy=LFU)
    hist = [[a, c], [a, c], [a], [a], [a, b, c]]
    for t, ks in enumerate(hist):
        _drive(o, t, [ks])
    vk, _ = o.victims(0)
    counts = dict(zip(*[o.dump_cache(0)[x].tolist() for x in ("keys", "count")]))
    assert counts == {a: 5, c: 3}
    assert vk.tolist() == [b], ex["cite"]
    # LRU touches {a:10, b:3, c:7} resident, a new key d at t=11 overflows capacity 3 -> evict b
    ex = golden["evict_overflow"][1]
    o = Oracle(R=16, D=0, C=3, s=S_INF, policy=LRU)
    for t, ks in [(3, [b]), (7, [c]), (10, [a]), (11, [d])]:
        _drive(o, t, [ks])
    assert o.victims(0)[0].tolist() == [b], ex["cite"]
    # LFU tie {a:2, b:2}, capacity 1 -> evict a (smaller key)
    ex = golden["evict_overflow"][2]
    o = Oracle(R=16, D=0, C=1, s=S_INF, policy=LFU)
    _drive(o, 0, [[a]])
    _drive(o, 1, [[b]])          # evicts a (count 1) vs b (count 1): tie -> a
    _drive(o, 2, [[a, b]])       # counts a:2, b:2, one over capacity -> a
    assert o.victims(0)[0].tolist() == [a], ex["cite"]


# ----------------------------------------------------------------------------- closed forms, N = 1
@pytest.mark.parametrize("s", [0, 1, 3, 10])
def test_single_worker_sync_period(s):
    """P5: with N=1, c_g only moves by this worker's own pushes, so a key read
    every iteration is synced exactly every s+1 iterations and EXP2 never occurs."""
    k = 4
    o = Oracle(R=8, D=0, C=8, s=s)
    st = []
    for t in range(40):
        _drive(o, t, [[k]])
        st.append(int(o.lookup_log(0)["status"][0]))
    assert st[0] == MISS
    for t in range(1, 40):
        assert st[t] == (EXP1 if t % (s + 1) == 0 else HIT), (t, st)
    assert o.stats(0)["exp2"] == 0


def _no_cache_sgd(keys_per_t, grads_per_t, D):
    """Plain sequential SGD on an uncached table (Eq. 2 for
    N=1 and the embedding update of Alg. 3): W_k += fl(-lr * sum_pos G)."""
    W = {}
    outs = []
    for keys, G in zip(keys_per_t, grads_per_t):
        for k in set(keys):
            if k not in W:
                W[k] = np.array([init_value(INIT_SEED, k, d) for d in range(D)], np.float32)
        outs.append(np.stack([W[k].copy() for k in keys]))
        for k in sorted(set(keys)):
            acc = np.zeros(D, np.float32)
            for p, kk in enumerate(keys):
                if kk == k:
                    acc = (acc + G[p]).astype(np.float32)
            W[k] = (W[k] + (F32(-LR) * acc).astype(np.float32)).astype(np.float32)
    return W, outs


@pytest.mark.parametrize("C", [3, 10, 64])
def test_s0_single_worker_equals_no_cache_sgd(C):
    """P6: N=1, s=0 is bit-exact sequential SGD without a cache, for any C."""
    rng = np.random.default_rng(C)
    R, D, T = 64, 4, 40
    keys_t = [list(rng.integers(0, R, size=rng.integers(1, 12))) for _ in range(T)]
    grads_t = [rnd_grads(rng, len(k), D) for k in keys_t]
    o = Oracle(R=R, D=D, C=C, s=0)
    outs = []
    for t in range(T):
        outs.append(o.lookup(t, [keys_t[t]])[0])
        o.update([grads_t[t]], LR)
    o.flush()
    W, ref_outs = _no_cache_sgd(keys_t, grads_t, D)
    for a, b in zip(outs, ref_outs):
        assert np.array_equal(a, b)
    ks = sorted(W)
    rows, _ = o.read_global(ks)
    assert np.array_equal(rows, np.stack([W[k] for k in ks]))


@pytest.mark.parametrize("N", [1, 2, 3])
def test_s0_never_valid_hit(N):
    """P6b: with s=0 every re-access is EXP1 (installed then written in the same iteration)."""
    rng = np.random.default_rng(N)
    o = Oracle(R=20, D=0, C=6, s=0, N=N)
    for t in range(60):
        ks = [list(rng.integers(0, 20, size=rng.integers(0, 8))) for _ in range(N)]
        _drive(o, t, ks)
    for i in range(N):
        st = o.stats(i)
        assert st["hits"] == 0 and st["exp2"] == 0 and st["exp1"] > 0


@pytest.mark.parametrize("N", [1, 3])
def test_unbounded_staleness_full_cache_cold_misses_only(N):
    """P7 / S:705: s=inf and C >= R: each key misses exactly once per worker;
    nothing is pushed until het_sync."""
    rng = np.random.default_rng(7)
    R = 30
    o = Oracle(R=R, D=0, C=R, s=S_INF, N=N)
    seen = [set() for _ in range(N)]
    for t in range(50):
        ks = [list(rng.integers(0, R, size=rng.integers(0, 10))) for _ in range(N)]
        _drive(o, t, ks)
        for i in range(N):
            seen[i] |= set(ks[i])
    for i in range(N):
        st = o.stats(i)
        assert st["misses"] == len(seen[i])
        assert st["evictions"] == 0 and st["dirty_pushes"] == 0
        assert st["hits"] == st["unique"] - st["misses"]
    _, cg = o.read_global(np.arange(R))
    assert (cg == 0).all()
    o.flush()
    _, cg = o.read_global(np.arange(R))
    assert cg.max() > 0


def test_capacity_after_every_update():
    """P9 / S:294: |cache| <= C after every Write."""
    rng = np.random.default_rng(3)
    for policy in (LFU, LRU):
        o = Oracle(R=50, D=0, C=7, s=2, policy=policy, N=2)
        for t in range(80):
            ks = [list(rng.integers(0, 50, size=rng.integers(0, 12))) for _ in range(2)]
            _drive(o, t, ks)
            assert o.cache_size(0) <= 7 and o.cache_size(1) <= 7


# ----------------------------------------------------------------------------- conservation
@pytest.mark.parametrize("N,s,C", [(1, 3, 5), (2, 1, 8), (3, 10, 4)])
def test_conservation_after_flush(N, s, C):
    """P11 / S:159: after het_sync every global row = W0 + sum of all deltas
    any worker ever produced (1e-5 abs; exact order differs by worker)."""
    rng = np.random.default_rng(11 + N)
    R, D = 25, 3
    o = Oracle(R=R, D=D, C=C, s=s, N=N)
    total = {}
    for t in range(60):
        ks = [list(rng.integers(0, R, size=rng.integers(0, 9))) for _ in range(N)]
        gs = [rnd_grads(rng, len(k), D) for k in ks]
        o.lookup(t, ks)
        o.update(gs, LR)
        for i in range(N):
            for k in sorted(set(ks[i])):
                acc = np.zeros(D, np.float32)
                for p, kk in enumerate(ks[i]):
                    if kk == k:
                        acc = (acc + gs[i][p]).astype(np.float32)
                total[k] = total.get(k, 0.0) + (F32(-LR) * acc).astype(np.float64)
    o.flush()
    ks = sorted(total)
    rows, _ = o.read_global(ks)
    for j, k in enumerate(ks):
        w0 = np.array([init_value(INIT_SEED, k, d) for d in range(D)], np.float64)
        assert np.abs(rows[j] - (w0 + total[k])).max() <= 1e-5


# ----------------------------------------------------------------------------- read-my-updates
def test_read_my_updates():
    """P12 / P:478-480: after a Write, the next Read of a valid hit returns exactly fl(v + delta)."""
    rng = np.random.default_rng(5)
    D = 4
    o = Oracle(R=10, D=D, C=10, s=S_INF)
    keys = [1, 2, 2, 5]
    out0 = o.lookup(0, [keys])[0]
    G = rnd_grads(rng, 4, D)
    o.update([G], LR)
    out1 = o.lookup(1, [keys])[0]
    assert (o.lookup_log(0)["status"] == HIT).all()
    for p, k in enumerate(keys):
        acc = np.zeros(D, np.float32)
        for q, kk in enumerate(keys):
            if kk == k:
                acc = (acc + G[q]).astype(np.float32)
        assert np.array_equal(out1[p], (out0[p] + (F32(-LR) * acc).astype(np.float32)).astype(np.float32))


# ----------------------------------------------------------------------------- Lemma 1
@pytest.mark.parametrize("s", [1, 2, 5])
def test_lemma1_bounds_at_read_instants(s):
    """P8 / Lemma 1: at each read, a valid hit satisfies
    cs <= cg_obs, cc <= cs + s and cg_obs <= cc + s; replicas validated in the
    same read differ by at most 2s."""
    rng = np.random.default_rng(100 + s)
    N, R = 3, 6
    o = Oracle(R=R, D=0, C=3, s=s, N=N)
    checked = 0
    for t in range(400):
        before = [o.dump_cache(i) for i in range(N)]
        _, cg_obs = o.read_global(np.arange(R))
        ks = [list(rng.integers(0, R, size=rng.integers(0, 4))) for _ in range(N)]
        o.lookup(t, ks)
        valid = {}
        for i in range(N):
            log = o.lookup_log(i)
            bk = dict(zip(before[i]["keys"].tolist(), zip(before[i]["cs"].tolist(), before[i]["cc"].tolist())))
            for k, stt in zip(log["unique"].tolist(), log["status"].tolist()):
                if stt != HIT:
                    continue
                cs, cc = bk[k]
                g = int(cg_obs[k])
                assert cs <= g and cc <= cs + s and g <= cc + s
                valid.setdefault(k, []).append(cc)
                checked += 1
        for k, ccs in valid.items():
            assert max(ccs) - min(ccs) <= 2 * s
        o.update(None, LR)
    assert checked > 50


# ----------------------------------------------------------------------------- brute-force replay
def _replay_case(seed):
    rng = np.random.default_rng(seed)
    R = int(rng.integers(2, 65))
    D = int(rng.integers(1, 5))
    N = int(rng.integers(1, 4))
    s = [0, 1, 3, S_INF][int(rng.integers(0, 4))]
    C = int(rng.integers(1, R + 1))
    policy = int(rng.integers(0, 2))
    persist = int(rng.integers(0, 2))
    return rng, R, D, N, s, C, policy, persist


@pytest.mark.parametrize("seed", range(40))
def test_brute_force_replay(seed):
    """P14: the oracle and the independent brute-force implementation agree
    bit-exactly on outs, statuses, victims and global rows."""
    rng, R, D, N, s, C, policy, persist = _replay_case(seed)
    o = Oracle(R=R, D=D, C=C, s=s, policy=policy, N=N, lfu_persist=persist)
    b = Brute(R=R, D=D, C=C, s=s, policy=policy, N=N, lfu_persist=persist)
    names = {HIT: "HIT", EXP1: "EXP1", EXP2: "EXP2", MISS: "MISS"}
    for t in range(30):
        ks = [list(rng.integers(0, R, size=rng.integers(0, 10))) for _ in range(N)]
        gs = [rnd_grads(rng, len(k), D) for k in ks]
        oo = o.lookup(t, ks)
        bo = b.lookup(t, ks)
        for i in range(N):
            assert np.array_equal(oo[i], bo[i])
            log = o.lookup_log(i)
            assert log["unique"].tolist() == b.logs[i]["uniq"]
            assert [names[x] for x in log["status"].tolist()] == b.logs[i]["status"]
        o.update(gs, LR)
        b.update(gs, LR)
        for i in range(N):
            vk, vd = o.victims(i)
            assert list(zip(vk.tolist(), vd.astype(bool).tolist())) == b.victims[i]
            c = o.dump_cache(i)
            assert c["keys"].tolist() == sorted(b.caches[i])
            for j, k in enumerate(c["keys"].tolist()):
                e = b.caches[i][k]
                assert np.array_equal(c["v"][j], np.array(e["v"], np.float32))
                assert (int(c["cs"][j]), int(c["cc"][j])) == (e["cs"], e["cc"])
    o.flush()
    b.flush()
    rows, cg = o.read_global(np.arange(R))
    for k in range(R):
        br, bcg = b.global_row(k)
        assert np.array_equal(rows[k], br) and int(cg[k]) == bcg


# ----------------------------------------------------------------------------- light-LFU (R27)
@pytest.mark.parametrize("seed", range(24))
def test_brute_force_replay_light_lfu(seed):
    """P14 for light-LFU: oracle == brute force on random tiny traces with
    small promotion thresholds (pins happen, the floor(C/2) cap binds)."""
    rng = np.random.default_rng(1000 + seed)
    R = int(rng.integers(2, 40))
    D = int(rng.integers(1, 4))
    N = int(rng.integers(1, 4))
    s = [0, 1, 3, S_INF][int(rng.integers(0, 4))]
    C = int(rng.integers(1, R + 1))
    persist = int(rng.integers(0, 2))
    thr = int(rng.integers(1, 5))
    o = Oracle(R=R, D=D, C=C, s=s, policy=LIGHT_LFU, N=N, lfu_persist=persist, pin_threshold=thr)
    b = Brute(R=R, D=D, C=C, s=s, policy=2, N=N, lfu_persist=persist, pin_thr=thr)
    names = {HIT: "HIT", EXP1: "EXP1", EXP2: "EXP2", MISS: "MISS"}
    pinned_seen = 0
    for t in range(40):
        ks = [list(rng.integers(0, R, size=rng.integers(0, 12))) for _ in range(N)]
        gs = [rnd_grads(rng, len(k), D) for k in ks]
        oo = o.lookup(t, ks)
        bo = b.lookup(t, ks)
        for i in range(N):
            assert np.array_equal(oo[i], bo[i])
            log = o.lookup_log(i)
            assert [names[x] for x in log["status"].tolist()] == b.logs[i]["status"]
        o.update(gs, LR)
        b.update(gs, LR)
        for i in range(N):
            vk, vd = o.victims(i)
            assert list(zip(vk.tolist(), vd.astype(bool).tolist())) == b.victims[i]
            c = o.dump_cache(i)
            pins = {k for k, tk in zip(c["keys"].tolist(), c["tick"].tolist()) if tk == PINNED}
            assert pins == b.pinned[i] and len(pins) <= C // 2
            pinned_seen += len(pins)
            for j, k in enumerate(c["keys"].tolist()):
                assert np.array_equal(c["v"][j], np.array(b.caches[i][k]["v"], np.float32))
                assert int(c["count"][j]) == (b.counts[i].get(k, 0) if persist else b.caches[i][k]["own"])
    o.flush()
    b.flush()
    rows, cg = o.read_global(np.arange(R))
    for k in range(R):
        br, bcg = b.global_row(k)
        assert np.array_equal(rows[k], br) and int(cg[k]) == bcg
    if C >= 2:
        assert pinned_seen > 0


def test_light_lfu_three_gets_promote():
    """SPEC S:289 vector: LightLFU threshold=3 -- three gets promote the entry;
    a pinned entry is never a victim and its count stops."""
    o = Oracle(R=10, D=1, C=2, s=S_INF, policy=LIGHT_LFU, pin_threshold=3)
    for t in range(3):
        o.lookup(t, [[5]])
        o.update(None, LR)
        c = o.dump_cache(0)
        assert (int(c["tick"][0]) == PINNED) == (t == 2)
    # keys 1 and 2 have count 1 < count(5) = 3 but 5 is pinned: the overflow
    # victims are chosen among the unpinned only, smallest (count, key) first
    for t in range(3, 6):
        o.lookup(t, [[5, 1, 2]])
        o.update(None, LR)
    c = o.dump_cache(0)
    assert 5 in c["keys"].tolist()
    assert int(c["count"][c["keys"].tolist().index(5)]) == 3      # no maintenance after the pin


def test_light_lfu_miss_rate_close_to_lfu():
    """light-LFU's miss rate stays within 2 percentage points of
    exact LFU on the same Zipf trace (P:632 'similar miss rate')."""
    from workload import gen
    cards = gen.scaled_cards(20000)
    rates = {}
    for pol in (LFU, LIGHT_LFU):
        o = Oracle(R=20000, D=0, C=2000, s=S_INF, policy=pol, pin_threshold=64)
        for t in range(400):
            o.lookup(t, [gen.criteo_keys(0, t, 1, 128, cards)[0].numpy()], want_out=False)
            o.update(None, LR)
            if t == 199:
                s0 = o.stats(0)
        s1 = o.stats(0)
        rates[pol] = (s1["misses"] - s0["misses"]) / (s1["unique"] - s0["unique"])
    assert abs(rates[LFU] - rates[LIGHT_LFU]) <= 0.02, rates


# ----------------------------------------------------------------------------- init (R14)
def test_init_rows_exact_in_range_never_negative_zero():
    from oracle.oracle import w0
    for k in [0, 1, 2, 999, 33762576]:
        for d in range(0, 128, 17):
            v = w0(k, d)
            assert v == init_value(INIT_SEED, k, d)
            assert -2.0 ** -7 <= v < 2.0 ** -7
            assert not (v == 0.0 and math.copysign(1.0, v) < 0)
            assert v * 2 ** 30 == int(v * 2 ** 30)
