"""Profiling driver: fill the WDL cache, then run K steps between
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees only the
steady-state kernels of the hot path.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python tools/prof_step.py --steps 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--fill", type=int, default=6500)
    ap.add_argument("--policy", default="LFU")
    ap.add_argument("--scale", action="store_true", help="BASELINE configs[4] per GPU: 3M rows, D = 4096")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, D = args.batch, (4096 if args.scale else 128)
    n = B * 26
    cards = gen.scaled_cards(3_000_000) if args.scale else gen.cards_for("criteo")
    R = sum(cards)
    pol = het.HET_LFU if args.policy == "LFU" else het.HET_LRU
    c = het.HetCache(R, D, 0.1, 100, pol, max_keys_per_call=n)
    fill = args.fill * 128 // B
    t = 0
    g = gen.grads(0, 0, n, D, device=dev)
    while t < fill:
        T = min(500, fill - t)
        keys = gen.criteo_keys(0, t, T, B, cards, device=dev)
        for j in range(T):
            c.lookup(keys[j], t)
            c.update(keys[j], g, 0.01)
            t += 1
    keys = gen.criteo_keys(0, t, args.steps, B, cards, device=dev)
    grads = [gen.grads(0, t + j, n, D, device=dev) for j in range(args.steps)]
    out = torch.empty((n, D), device=dev)
    torch.cuda.synchronize()
    print("resident", c.stats()["resident"], flush=True)
    torch.cuda.cudart().cudaProfilerStart()
    for j in range(args.steps):
        c.lookup(keys[j], t + j, out=out)
        c.update(keys[j], grads[j], 0.01)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("stats", c.stats(), flush=True)


if __name__ == "__main__":
    main()
