"""A small run of the hot path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): toy config (BASELINE configs[0]) at N = 1 on the fused
and the per-phase kernels, and a loopback group of N = 2 workers on one GPU
(the exchange round phase by phase, pushes, flush, Eq. 2).  Exits 0 on
success; the sanitizer's own report decides clean or not.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402

T = int(os.environ.get("SAN_STEPS", "12"))
R, D, cards = 1000, 8, gen.cards_for("toy")


def keys_of(i, t):
    return gen.criteo_keys(i, t, 1, 128, cards)[0].cuda()


def n1(policy):
    c = het.HetCache(R, D, 0.1, 3, policy, max_keys_per_call=4096)
    for t in range(T):
        k = keys_of(0, t)
        c.lookup(k, t)
        c.update(k, gen.grads(0, t, k.numel(), D).cuda(), 0.01)
    c.evict(keys_of(0, 0)[:40])
    c.sync()
    c.close()


def loopback():
    g = het.HetGroup(2, R, D, 0.1, 3, het.HET_LFU, max_keys_per_call=4096, dense_max=1024)
    for t in range(T):
        ks = [keys_of(i, t) for i in range(2)]
        g.lookup(ks, t)
        g.update(ks, [gen.grads(i, t, k.numel(), D).cuda() for i, k in enumerate(ks)], 0.01)
    g.evict([k[:30] for k in ks])
    g.dense_allreduce([torch.arange(1000, device="cuda", dtype=torch.float32) * (i + 1) for i in range(2)])
    g.sync()
    g.close()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    n1(het.HET_LFU)
    n1(het.HET_LRU)
    os.environ["HET_NO_FUSED"] = "1"
    n1(het.HET_LFU)
    del os.environ["HET_NO_FUSED"]
    loopback()
    torch.cuda.synchronize()
    print("SANITIZE_RUN_OK", flush=True)
