"""NEXT-4: end-to-end training of WDL-, DCN- and
GraphSAGE-shaped models (the paper's workloads, Table 3) whose
sparse embeddings live in the HET cache, on teacher-labelled synthetic data.
The dense towers are plain PyTorch; every embedding row moves through the
C-ABI (`het_lookup` -> forward/backward -> `het_update` with the rows'
gradients), and the dense gradients are synchronised with
`het_dense_allreduce` (Eq. 2).  One process per GPU (torchrun),
the table hash-sharded over the GPUs.

Models (--model):
  wdl        Wide & Deep over 26 Criteo-shaped fields: deep MLP + wide linear
  dcn        Deep & Cross over the same fields: 3 cross layers
             x_{l+1} = x0 * (x_l . w_l) + b_l + x_l beside the deep MLP
  graphsage  GraphSAGE over Reddit-shaped node ids: per step B seed
             nodes with 10 sampled neighbours each and 10 of each of those
             (B * 111 ids, all distinct: the all-unique dedup regime), node
             features are HET embeddings, two mean-aggregation SAGE layers

The paper's convergence experiments (Table 3: AUC vs staleness s)
need Criteo itself and are out of scope; this reproduces the *pattern* on a
synthetic task: with s in {0, 10, 100, inf} the progressive AUC stays close to
the s = 0 run at moderate s while the embedding bytes on the wire drop.

Labels: a fixed teacher, y ~ Bernoulli(sigmoid(sum_f theta[key_f] + b0)),
theta[key] from a counter hash of the key (workload.gen.mix64), so every
worker draws labels from the same ground truth.

    python examples/train.py --model wdl --staleness 10 --steps 600
    torchrun --nproc-per-node 2 examples/train.py --model dcn --staleness 10 --steps 600
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


def labels(keys: torch.Tensor, F: int, rank: int, t: int, graph: bool = False) -> torch.Tensor:
    if graph:   # a seed's label from its own id and its sampled 1-hop neighbourhood
        f = SAGE.FAN
        B = keys.numel() // (1 + f + f * f)
        own = teacher_logit(keys[:B], 1)
        nbr = teacher_logit(keys[B:B + B * f], f)
        p = torch.sigmoid(own + 0.5 * nbr)
    else:
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


class DCN(torch.nn.Module):
    """DCN-shaped dense part: cross network (explicit feature crosses) beside a deep MLP."""

    def __init__(self, F: int, D: int, layers: int = 3):
        super().__init__()
        d = F * D
        self.w = torch.nn.ParameterList([torch.nn.Parameter(torch.randn(d) * d ** -0.5) for _ in range(layers)])
        self.b = torch.nn.ParameterList([torch.nn.Parameter(torch.zeros(d)) for _ in range(layers)])
        self.deep = torch.nn.Sequential(torch.nn.Linear(d, 256), torch.nn.ReLU(), torch.nn.Linear(256, 128),
                                        torch.nn.ReLU())
        self.out = torch.nn.Linear(d + 128, 1)

    def forward(self, x0):
        x = x0
        for w, b in zip(self.w, self.b):
            x = x0 * (x @ w).unsqueeze(1) + b + x
        return self.out(torch.cat([x, self.deep(x0)], 1)).squeeze(1)


class SAGE(torch.nn.Module):
    """GraphSAGE-shaped dense part over a sampled 2-hop tree per seed (fan-out 10):
    h1(v) = relu(W1 [e(v) || mean e(children)]) for the seed and its 1-hop nodes,
    h2(seed) = relu(W2 [h1(seed) || mean h1(1-hop)]), logit = w . h2."""

    FAN = 10

    def __init__(self, D: int, H: int = 64):
        super().__init__()
        self.l1 = torch.nn.Linear(2 * D, H)
        self.l2 = torch.nn.Linear(2 * H, H)
        self.out = torch.nn.Linear(H, 1)

    def forward(self, e):
        B = e.shape[0] // (1 + self.FAN + self.FAN * self.FAN)
        f = self.FAN
        seed, hop1, hop2 = e[:B], e[B:B + B * f].view(B, f, -1), e[B + B * f:].view(B, f, f, -1)
        h1_seed = torch.relu(self.l1(torch.cat([seed, hop1.mean(1)], 1)))
        h1_hop1 = torch.relu(self.l1(torch.cat([hop1, hop2.mean(2)], 2)))
        h2 = torch.relu(self.l2(torch.cat([h1_seed, h1_hop1.mean(1)], 1)))
        return self.out(h2).squeeze(1)


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
    ap.add_argument("--model", default="wdl", choices=["wdl", "dcn", "graphsage"])
    ap.add_argument("--staleness", type=int, default=10, help="staleness threshold s (-1 = infinity)")
    ap.add_argument("--steps", type=int, default=600)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--D", type=int, default=16)
    ap.add_argument("--batch", type=int, default=0, help="samples per worker-iteration (0: 512, graphsage 128)")
    ap.add_argument("--cache-frac", type=float, default=0.1)
    ap.add_argument("--lr", type=float, default=0.05, help="dense SGD step")
    ap.add_argument("--emb-lr", type=float, default=0.0,
                    help="embedding SGD step (mean-loss gradients are 1/B per row; 0: 5, graphsage 200)")
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
    graph = args.model == "graphsage"
    D, B = args.D, args.batch or (128 if graph else 512)
    emb_lr = args.emb_lr or (200.0 if graph else 5.0)
    F = 1 + SAGE.FAN + SAGE.FAN * SAGE.FAN if graph else 26   # ids per sample
    rows = min(args.rows, gen.REDDIT_ROWS) if graph else args.rows
    cards = None if graph else gen.scaled_cards(rows)
    s = het.HET_S_INF if args.staleness < 0 else args.staleness
    cache = het.HetCache(rows, D, args.cache_frac, s, het.HET_LFU, rank=rank, world=world,
                         unique_id=uid, max_keys_per_call=B * F)
    torch.manual_seed(0)                              # same dense init on every worker
    tower = {"wdl": lambda: Tower(F, D), "dcn": lambda: DCN(F, D), "graphsage": lambda: SAGE(D)}[args.model]().to(dev)
    params = list(tower.parameters())
    flat = torch.zeros(sum(p.numel() for p in params), device=dev)
    lossf = torch.nn.BCEWithLogitsLoss()
    preds, ys, losses = [], [], []
    if graph:   # Reddit-shaped: B * 111 distinct node ids per worker-iteration (Zipf(1.0) over the nodes)
        keys_all = None
    else:
        keys_all = gen.criteo_keys(rank, 0, args.steps, B, cards, device=dev)
    torch.cuda.synchronize()
    t0 = time.time()
    for t in range(args.steps):
        keys = gen.reddit_keys(rank, t, B * F, rows, device=dev) if graph else keys_all[t]
        y = labels(keys, F, rank, t, graph)
        emb = cache.lookup(keys, het.HET_CLOCK_AUTO)           # Het.Read (Alg. 2)
        x = (emb if graph else emb.view(B, F * D)).requires_grad_(True)
        logit = tower(x)
        loss = lossf(logit, y)
        for p in params:
            p.grad = None
        loss.backward()
        cache.update(keys, x.grad.reshape(B * F, D), emb_lr)   # Het.Write (Alg. 3)
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
    res = {"model": args.model, "s": "inf" if args.staleness < 0 else args.staleness, "n_gpus": world,
           "steps": args.steps, "batch_per_gpu": B, "rows": rows, "D": D, "progressive_auc": auc(yy.cpu().numpy(), pr.cpu().numpy()),
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
