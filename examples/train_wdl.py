"""NEXT-4: end-to-end training of a WDL-shaped model whose
sparse embeddings live in the HET cache, on teacher-labelled synthetic
Criteo-shaped data.  The dense tower is plain PyTorch; every embedding
row moves through the C-ABI (`het_lookup` -> forward/backward ->
`het_update` with the rows' gradients), and the dense gradients are
synchronised with `het_dense_allreduce` (Eq. 2).  One process per
GPU (torchrun), the table hash-sharded over the GPUs.

The paper's convergence experiments (Table 3: AUC vs staleness s)
need Criteo itself and are out of scope; this reproduces the *pattern* on a
synthetic task: with s in {0, 10, 100, inf} the progressive AUC stays close to
the s = 0 run at moderate s while the embedding bytes on the wire drop.

Labels: a fixed teacher, y ~ Bernoulli(sigmoid(sum_f theta[key_f] + b0)),
theta[key] from a counter hash of the key (workload.gen.mix64), so every
worker draws labels from the same ground truth.

    python examples/train_wdl.py --s 10 --steps 600
    torchrun --nproc-per-node 2 examples/train_wdl.py --s 10 --steps 600
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2112_07221_b200 import het  # noqa: E402
from workload import gen  # noqa: E402


def teacher_logit(keys: torch.Tensor, F: int) -> torch.Tensor:
    """sum over the sample's fields of theta[key], theta in [-1.5, 1.5) per key."""
    h = gen.mix64(keys ^ 0x5EED7EAC4E5)
    theta = gen.uniform(h).to(torch.float32) * 3.0 - 1.5
    return theta.view(-1, F).sum(1) * (2.0 / F ** 0.5)


def labels(keys: torch.Tensor, F: int, rank: int, t: int) -> torch.Tensor:
    p = torch.sigmoid(teacher_logit(keys, F))
    u = gen.uniform(gen.stream(gen.SEED + 7, rank, t, torch.arange(p.numel(), device=keys.device)))
    return (u.to(torch.float32) < p).to(torch.float32)


class Tower(torch.nn.Module):
    """WDL-shaped dense part: deep MLP over the concatenated field embeddings
    plus a wide linear term."""

    def __init__(self, F: int, D: int):
        super().__init__()
        self.deep = torch.nn.Sequential(torch.nn.Linear(F * D, 256), torch.nn.ReLU(),
                                        torch.nn.Linear(256, 128), torch.nn.ReLU(),
                                        torch.nn.Linear(128, 1))
        self.wide = torch.nn.Linear(F * D, 1)

    def forward(self, x):
        return (self.deep(x) + self.wide(x)).squeeze(1)


def auc(y: np.ndarray, p: np.ndarray) -> float:
    """ROC AUC by the rank statistic (ties averaged)."""
    order = np.argsort(p, kind="mergesort")
    ranks = np.empty(len(p), np.float64)
    ps = p[order]
    i = 0
    while i < len(ps):
        j = i
        while j + 1 < len(ps) and ps[j + 1] == ps[i]:
            j += 1
        ranks[order[i:j + 1]] = (i + j) / 2.0 + 1.0
        i = j + 1
    pos = y > 0.5
    npos, nneg = pos.sum(), (~pos).sum()
    return float((ranks[pos].sum() - npos * (npos + 1) / 2.0) / max(npos * nneg, 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--staleness", type=int, default=10, help="staleness threshold s (-1 = infinity)")
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--D", type=int, default=16)
    ap.add_argument("--batch", type=int, default=512)
    ap.add_argument("--cache-frac", type=float, default=0.1)
    ap.add_argument("--lr", type=float, default=0.05, help="dense SGD step")
    ap.add_argument("--emb-lr", type=float, default=5.0, help="embedding SGD step (mean-loss gradients are 1/B per row)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    uid = None
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
        obj = [het.het_get_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        uid = obj[0]
    F, D, B = 26, args.D, args.batch
    cards = gen.scaled_cards(args.rows)
    s = het.HET_S_INF if args.staleness < 0 else args.staleness
    cache = het.HetCache(args.rows, D, args.cache_frac, s, het.HET_LFU, rank=rank, world=world,
                         unique_id=uid, max_keys_per_call=B * F)
    torch.manual_seed(0)                              # same dense init on every worker
    tower = Tower(F, D).to(dev)
    params = list(tower.parameters())
    flat = torch.zeros(sum(p.numel() for p in params), device=dev)
    lossf = torch.nn.BCEWithLogitsLoss()
    preds, ys, losses = [], [], []
    keys_all = gen.criteo_keys(rank, 0, args.steps, B, cards, device=dev)
    torch.cuda.synchronize()
    t0 = time.time()
    for t in range(args.steps):
        keys = keys_all[t]
        y = labels(keys, F, rank, t)
        emb = cache.lookup(keys, het.HET_CLOCK_AUTO)           # Het.Read (Alg. 2)
        x = emb.view(B, F * D).requires_grad_(True)
        logit = tower(x)
        loss = lossf(logit, y)
        for p in params:
            p.grad = None
        loss.backward()
        cache.update(keys, x.grad.view(B * F, D), args.emb_lr)   # Het.Write (Alg. 3)
        off = 0                                                # Eq. 2: mean of the dense grads
        for p in params:
            flat[off:off + p.numel()].copy_(p.grad.view(-1))
            off += p.numel()
        het.het_dense_allreduce(cache.h, flat, flat.numel())
        off = 0
        with torch.no_grad():
            for p in params:
                p.add_(flat[off:off + p.numel()].view_as(p), alpha=-args.lr)
                off += p.numel()
        if t >= args.steps // 2:                               # progressive validation
            preds.append(torch.sigmoid(logit.detach()))
            ys.append(y)
            losses.append(loss.detach())
    torch.cuda.synchronize()
    dt = time.time() - t0
    st = cache.stats()
    pr = torch.cat(preds)
    yy = torch.cat(ys)
    if world > 1:                                              # pool the validation samples
        gp = [torch.empty_like(pr) for _ in range(world)]
        gy = [torch.empty_like(yy) for _ in range(world)]
        torch.distributed.all_gather(gp, pr)
        torch.distributed.all_gather(gy, yy)
        pr, yy = torch.cat(gp), torch.cat(gy)
    res = {"s": "inf" if args.staleness < 0 else args.staleness, "n_gpus": world, "steps": args.steps, "batch_per_gpu": B,
           "rows": args.rows, "D": D, "progressive_auc": auc(yy.cpu().numpy(), pr.cpu().numpy()),
           "loss_second_half": float(torch.stack(losses).mean()),
           "samples_per_s": B * world * args.steps / dt,
           "emb_bytes_tx_per_step": (st["bytes_emb_tx"] + st["bytes_clock_tx"]) / args.steps,
           "misses": st["misses"], "exp1": st["exp1"], "exp2": st["exp2"], "hits": st["hits"]}
    cache.sync()
    cache.close()
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
