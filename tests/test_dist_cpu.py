"""world_size-2 gloo test (CPU) of the multi-GPU exchange design.

tests/dist_model.py runs one worker per process with its shard of the global
table and exchanges the same records the CUDA peer-memory exchange sends
(eviction pushes carried by the next round, clock check folded into the fetch
round, per-row source-ordered owner apply).  Each rank checks its outputs,
statuses, victims and, after the flush, its shard against the N-worker
lock-step oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Oracle, capacity, HIT, EXP1, EXP2, MISS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, policy, s, frac, T, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from dist_model import Rank
        from workload import gen
        R, D, lr = 300, 4, 0.01
        cards = [12] * 13 + [11] * 13   # 299 rows... pad below
        cards[0] += R - sum(cards)
        C = capacity(frac, R)
        o = Oracle(R=R, D=D, C=C, s=s, policy=policy, N=world)
        w = Rank(R, D, C, s, rank, world, policy)
        names = {HIT: "HIT", EXP1: "EXP1", EXP2: "EXP2", MISS: "MISS"}
        for t in range(T):
            keys = [gen.criteo_keys(i, t, 1, 8, cards)[0].numpy() for i in range(world)]
            if t % 5 == 2:
                keys[1 % world] = keys[1 % world][:3]
            grads = [gen.grads(i, t, k.size, D).numpy() for i, k in enumerate(keys)]
            oo = o.lookup(t, keys)
            out, st, uniq = w.lookup(t, keys[rank])
            assert np.array_equal(out, oo[rank]), t
            log = o.lookup_log(rank)
            assert uniq == log["unique"].tolist(), t
            assert st == [names[x] for x in log["status"].tolist()], (t, st)
            o.update(grads, lr)
            w.update(grads[rank], lr)
            vk, vd = o.victims(rank)
            assert sorted(w.victims) == sorted(zip(vk.tolist(), vd.astype(bool).tolist())), t
        o.flush()
        w.flush()
        owned = [k for k in range(R) if k % world == rank]
        rows, cg = o.read_global(owned)
        for j, k in enumerate(owned):
            assert np.array_equal(w._row(k), rows[j]) and w.cg.get(k, 0) == int(cg[j]), k
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("policy,s,frac", [(0, 2, 0.1), (1, 0, 0.05), (0, 0xFFFFFFFF, 0.2)])
def test_sharded_exchange_world2_gloo(policy, s, frac):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, policy, s, frac, 40, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", msg
