"""Distributed CPU model of the sharded exchange (one process per worker, gloo).

Each rank owns the global rows k with k mod N == rank and its own cache.  One
lookup is one exchange round, exactly as the CUDA peer-memory exchange
(paper_2112_07221_b200/csrc/het_p2p.cu) orders it: the eviction pushes of the
rank's previous update travel first, then this lookup's requests (hits that
passed condition (1) with their pending row, expired hits, misses); every
owner handles each row's records in source-rank order -- pushes (U4 of t-1),
condition (2) against c_g after them (L3), sync pushes (L4), responses (L5).
Messages are exchanged with all_gather_object over gloo.

Used by tests/test_dist_cpu.py to check the design of the multi-GPU path
against the N-worker oracle without GPUs.
"""
from __future__ import annotations

import numpy as np
import torch.distributed as dist

F32 = np.float32
S_INF = 0xFFFFFFFF
M64 = (1 << 64) - 1


def _fm(x):
    x &= M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M64
    x ^= x >> 31
    return x


def w0(seed0, key, d):
    h = _fm(_fm(_fm(int(seed0)) ^ int(key)) ^ int(d))
    return F32(((h >> 40) - (1 << 23)) / float(1 << 30))


class Rank:
    def __init__(self, R, D, C, s, rank, world, policy=0, seed0=2112072210):
        self.R, self.D, self.C, self.s = R, D, C, s
        self.rank, self.N, self.policy, self.seed0 = rank, world, policy, seed0
        self.W, self.cg = {}, {}          # owned rows only
        self.cache = {}                   # key -> dict(v, p, cs, cc, tick)
        self.count = {}
        self.pending = []                 # eviction pushes waiting for the next round
        self.victims = []

    def _row(self, k):
        if k not in self.W:
            self.W[k] = np.array([w0(self.seed0, k, d) for d in range(self.D)], np.float32)
        return self.W[k]

    def _round(self, requests):
        """requests: list of (key, kind, cc, row or None); kind in push/needq/exp1/miss."""
        N = self.N
        outbox = [[] for _ in range(N)]
        for rec in self.pending + requests:
            outbox[rec[0] % N].append(rec)
        self.pending = []
        inbox = [None] * N
        gathered = [None] * N
        dist.all_gather_object(gathered, outbox)
        for src in range(N):
            inbox[src] = gathered[src][self.rank]
        # owner: group by row, source order (pushes of a source precede its requests)
        rows = {}
        for src in range(N):
            for j, rec in enumerate(inbox[src]):
                rows.setdefault(rec[0], []).append((src, j, rec))
        answers = [dict() for _ in range(N)]
        for k, lst in rows.items():
            W = self._row(k)
            g = self.cg.get(k, 0)
            for src, j, (key, kind, cc, row) in lst:           # U4(t-1)
                if kind == "push":
                    W[:] = (W + row).astype(np.float32)
                    g = max(g, cc)
            valid = {}
            for src, j, (key, kind, cc, row) in lst:           # L3
                if kind == "needq":
                    valid[(src, j)] = g <= cc + self.s
            for src, j, (key, kind, cc, row) in lst:           # L4
                if kind in ("needq", "exp1") and not valid.get((src, j), False) and row is not None:
                    W[:] = (W + row).astype(np.float32)
                    g = max(g, cc)
            self.cg[k] = g
            for src, j, (key, kind, cc, row) in lst:           # L5
                if kind != "push":
                    answers[src][key] = (g, valid.get((src, j), False), W.copy())
        back = [None] * N
        dist.all_gather_object(back, answers)
        mine = {}
        for o in range(N):
            mine.update(back[o][self.rank])
        return mine

    def lookup(self, t, keys):
        keys = [int(k) for k in keys]
        uniq = sorted(set(keys))
        status, reqs = {}, []
        for k in uniq:
            e = self.cache.get(k)
            if e is None:
                status[k] = "MISS"
                reqs.append((k, "miss", 0, None))
                continue
            if self.s == S_INF:
                status[k] = "HIT"
                continue
            dirty = e["cc"] > e["cs"]
            if e["cc"] - e["cs"] > self.s:
                status[k] = "EXP1"
                reqs.append((k, "exp1", e["cc"], e["p"].copy() if dirty else None))
            else:
                status[k] = "NEEDQ"
                reqs.append((k, "needq", e["cc"], e["p"].copy() if dirty else None))
        ans = self._round(reqs)
        for k in uniq:
            if status[k] == "HIT":
                continue
            g, valid, row = ans[k]
            if status[k] == "NEEDQ":
                if valid:
                    status[k] = "HIT"
                    continue
                status[k] = "EXP2"
            old = self.cache.get(k)
            self.cache[k] = dict(v=row.copy(), p=np.zeros(self.D, np.float32), cs=g, cc=g,
                                 tick=old["tick"] if old else 0)
        for k in uniq:
            self.count[k] = self.count.get(k, 0) + 1
            self.cache[k]["tick"] = t
        self.last = (keys, uniq)
        out = np.stack([self.cache[k]["v"] for k in keys]) if keys else np.zeros((0, self.D), np.float32)
        return out, [status[k] for k in uniq], uniq

    def update(self, grads, lr):
        keys, uniq = self.last
        lr = F32(lr)
        for k in uniq:
            e = self.cache[k]
            acc = np.zeros(self.D, np.float32)
            for pos, kk in enumerate(keys):
                if kk == k:
                    acc = (acc + grads[pos]).astype(np.float32)
            delta = (F32(-lr) * acc).astype(np.float32)
            e["v"] = (e["v"] + delta).astype(np.float32)
            e["p"] = (e["p"] + delta).astype(np.float32)
            e["cc"] += 1
        self.victims = []
        while len(self.cache) > self.C:
            prim = (lambda k: self.count[k]) if self.policy == 0 else (lambda k: self.cache[k]["tick"])
            k = min(self.cache, key=lambda q: (prim(q), q))
            e = self.cache.pop(k)
            dirty = e["cc"] > e["cs"]
            self.victims.append((k, dirty))
            if dirty:
                self.pending.append((k, "push", e["cc"], e["p"].copy()))

    def flush(self):
        # deliver the last update's eviction pushes first (U4 precedes the flush:
        # the CUDA path drains them the same way before het_sync's flush)
        self._round([])
        reqs = []
        for k in sorted(self.cache):
            e = self.cache[k]
            if e["cc"] > e["cs"]:
                self.pending.append((k, "push", e["cc"], e["p"].copy()))
        self.cache = {}
        self._round(reqs)
