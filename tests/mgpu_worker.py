"""One rank of the multi-GPU parity run (launched by tests/test_gpu_multi.py).

Every rank runs the same N-worker lock-step oracle and checks its own worker
against it: gathered rows (1e-6 rel), unique keys and statuses (bit-exact),
victims (bit-exact), counters, and at the end the rows/clocks of the global
table shard it owns.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle.oracle import Oracle, capacity  # noqa: E402
from workload import gen  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    policy, s, frac, T = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    from paper_2112_07221_b200 import het
    obj = [het.het_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    # shape: toy (BASELINE configs[0] rows, D=8), reddit (configs[2]: 232,965 ids,
    # 14,208 distinct ids per worker-iteration -> the large-n exchange path),
    # wide (Criteo-shaped fields over 5,000 rows with 4 KB rows, D=1024)
    shape = sys.argv[5] if len(sys.argv) > 5 else "toy"
    pin = int(sys.argv[6]) if len(sys.argv) > 6 else 64      # light-LFU threshold (policy 2)
    lr = 0.01
    if shape == "reddit":
        R, D, n_max = gen.REDDIT_ROWS, 128, 14208
    elif shape == "wide":
        R, D, n_max, cards = 5000, 1024, 4096, gen.scaled_cards(5000)
    else:
        R, D, n_max, cards = 1000, 8, 4096, gen.cards_for("toy")
    g = het.HetCache(R, D, frac, s, policy, rank=rank, world=world, unique_id=obj[0], max_keys_per_call=n_max,
                     pin_threshold=pin, dense_max=2048)
    o = Oracle(R=R, D=D, C=capacity(frac, R), s=s, policy=policy, N=world, pin_threshold=pin)
    for t in range(T):
        if shape == "reddit":
            keys = [gen.reddit_keys(i, t, n_max).numpy() for i in range(world)]
        else:
            keys = [gen.criteo_keys(i, t, 1, 128, cards)[0].numpy() for i in range(world)]
        if t % 7 == 3:                        # ragged: some workers send fewer keys
            keys = [k[: (k.size // 33) * (i + 1)] for i, k in enumerate(keys)]
        grads = [gen.grads(i, t, k.size, D).numpy() for i, k in enumerate(keys)]
        kd = torch.from_numpy(keys[rank]).cuda()
        out = g.lookup(kd, t).cpu().numpy()
        oo = o.lookup(t, keys)
        np.testing.assert_allclose(out, oo[rank], rtol=1e-6, atol=1e-30)
        gl, ol = g.lookup_log(), o.lookup_log(rank)
        assert np.array_equal(gl["unique"], ol["unique"]), t
        assert np.array_equal(gl["status"], ol["status"]), (t, np.nonzero(gl["status"] != ol["status"]))
        g.update(kd, torch.from_numpy(grads[rank]).cuda(), lr)
        o.update(grads, lr)
        gk, gdirty = g.victims()
        ok, od = o.victims(rank)
        order = np.argsort(ok, kind="stable")
        assert np.array_equal(gk, ok[order]), t
        assert np.array_equal(gdirty, od[order]), t
    gs, os_ = g.stats(), o.stats(rank)
    for k in ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses", "evictions", "dirty_pushes"]:
        assert gs[k] == os_[k], (k, gs[k], os_[k])
    assert gs["bytes_emb_tx"] > 0
    if policy == 2:
        assert gs["pinned"] > 0
    g.sync()
    o.flush()
    owned = np.arange(rank, R, world, dtype=np.int64)
    gr, gcg = g.read_global(owned)
    orows, ocg = o.read_global(owned)
    assert np.array_equal(gcg, ocg)
    np.testing.assert_allclose(gr, orows, rtol=1e-6, atol=1e-30)
    # dense all-reduce (Eq. 2): mean over workers
    # (peer-memory one-shot mean; epochs reuse the two staging buffers; a
    # shorter call exercises the scalar tail; one beyond dense_max falls back to NCCL)
    for k, cnt in enumerate([1000, 1000, 998, 1000, 4096]):
        x = torch.arange(cnt, device="cuda", dtype=torch.float32) * (rank + 1) + k
        het.het_dense_allreduce(g.h, x, x.numel())
        torch.cuda.synchronize()
        want = torch.arange(cnt, device="cuda", dtype=torch.float32) * ((world + 1) / 2.0) + k
        assert torch.allclose(x, want, rtol=1e-6, atol=1e-6), (k, cnt)
    g.close()
    dist.barrier()
    if rank == 0:
        print(f"MGPU_OK world={world} shape={shape} policy={policy} s={s} frac={frac} exp2={os_['exp2']} "
              f"evictions={os_['evictions']}", flush=True)


if __name__ == "__main__":
    main()
