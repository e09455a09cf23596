"""Independent brute-force replay of HET's cache protocol (pin P14).

Written separately from oracle/het_oracle.cpp, in plain Python dicts and
lists, for tiny tables only: victims are found by a linear scan over every
resident entry, unique keys by sorted(set(...)), fp32 arithmetic by numpy
float32 scalars (IEEE round-to-nearest-even, no FMA).  It follows the paper:
Fetch, Evict, CheckValid, Alg. 2 Read
(P:486-504), Alg. 3 Write, under the lock-step reading R1 and
R2-R17 of DESIGN.md.  Agreement between this file and the C++ oracle on random
traces is the pin for row values the paper never prints (P15).
"""
from __future__ import annotations

import numpy as np

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


def init_value(seed0, key, d):
    """R14 initial row value, integer arithmetic then one exact scaling."""
    h = _fm(_fm(_fm(int(seed0)) ^ int(key)) ^ int(d))
    return F32(((h >> 40) - (1 << 23)) / float(1 << 30))


class Brute:
    def __init__(self, R, D, C, s, policy=0, N=1, lfu_persist=1, seed0=2112072210, pin_thr=64):
        """policy 0 LFU, 1 LRU, 2 light-LFU: a key whose LFU count
        reaches pin_thr is pinned (no more count updates, never a victim),
        keys taken in ascending order while fewer than C // 2 are pinned (R27)."""
        self.R, self.D, self.C, self.s, self.policy, self.N = R, D, C, s, policy, N
        self.pin_thr = pin_thr
        self.pinned = [set() for _ in range(N)]
        self.persist = lfu_persist
        self.seed0 = seed0
        self.W = {}      # key -> list of F32 (server rows, lazily initialised)
        self.cg = {}     # key -> global clock
        self.caches = [dict() for _ in range(N)]   # key -> dict(v, p, cs, cc, tick, own)
        self.counts = [dict() for _ in range(N)]   # persistent LFU counts
        self.logs = [None] * N
        self.victims = [[] for _ in range(N)]

    # ---------------------------------------------------------------- server
    def _row(self, k):
        if k not in self.W:
            self.W[k] = [init_value(self.seed0, k, d) for d in range(self.D)]
        return self.W[k]

    def _push(self, k, p, cc):
        row = self._row(k)
        for d in range(self.D):
            row[d] = F32(row[d] + p[d])
        self.cg[k] = max(self.cg.get(k, 0), cc)

    # ---------------------------------------------------------------- read
    def lookup(self, t, keys_list):
        s = self.s
        for i in range(self.N):
            keys = [int(k) for k in keys_list[i]]
            uniq = sorted(set(keys))
            pos_of = {k: [p for p in range(len(keys)) if keys[p] == k] for k in uniq}
            status = []
            for k in uniq:
                c = self.caches[i]
                if k not in c:
                    status.append("MISS")
                    continue
                e = c[k]
                if s == S_INF:
                    status.append("HIT")
                    continue
                # CheckValid, exactly the paper's two inequalities on unbounded ints
                ok1 = e["cc"] <= e["cs"] + s
                if not ok1:
                    status.append("EXP1")
                    continue
                ok2 = self.cg.get(k, 0) <= e["cc"] + s
                status.append("HIT" if ok2 else "EXP2")
            self.logs[i] = dict(keys=keys, uniq=uniq, pos_of=pos_of, status=status)
        # all sync pushes (worker order, key order) before any fetch
        for i in range(self.N):
            L = self.logs[i]
            for k, st in zip(L["uniq"], L["status"]):
                if st in ("EXP1", "EXP2"):
                    e = self.caches[i][k]
                    if e["cc"] > e["cs"]:
                        self._push(k, e["p"], e["cc"])
        for i in range(self.N):
            L = self.logs[i]
            for k, st in zip(L["uniq"], L["status"]):
                if st == "HIT":
                    continue
                old = self.caches[i].get(k)
                g = self.cg.get(k, 0)
                self.caches[i][k] = dict(v=list(self._row(k)), p=[F32(0.0)] * self.D, cs=g, cc=g,
                                         tick=old["tick"] if old else 0,
                                         own=old["own"] if (old and st != "MISS") else 0)
        for i in range(self.N):
            for k in self.logs[i]["uniq"]:
                if k in self.pinned[i]:
                    continue
                self.counts[i][k] = self.counts[i].get(k, 0) + 1
                self.caches[i][k]["own"] += 1
                self.caches[i][k]["tick"] = t
                if self.policy == 2 and self._prim(i, k) >= self.pin_thr and len(self.pinned[i]) < self.C // 2:
                    self.pinned[i].add(k)
        outs = []
        for i in range(self.N):
            keys = self.logs[i]["keys"]
            outs.append(np.array([self.caches[i][k]["v"] for k in keys], dtype=np.float32)
                        .reshape(len(keys), self.D))
        return outs

    # ---------------------------------------------------------------- write
    def _prim(self, i, k):
        e = self.caches[i][k]
        if self.policy in (0, 2):
            return self.counts[i].get(k, 0) if self.persist else e["own"]
        return e["tick"]

    def update(self, grads_list, lr):
        lr = F32(lr)
        pushes = [[] for _ in range(self.N)]
        for i in range(self.N):
            L = self.logs[i]
            G = grads_list[i]
            for k in L["uniq"]:
                e = self.caches[i][k]
                for d in range(self.D):
                    acc = F32(0.0)
                    for p in L["pos_of"][k]:          # ascending batch position
                        acc = F32(acc + F32(G[p][d]))
                    delta = F32(F32(-lr) * acc)
                    e["v"][d] = F32(e["v"][d] + delta)
                    e["p"][d] = F32(e["p"][d] + delta)
                e["cc"] += 1
            self.victims[i] = []
            while len(self.caches[i]) > self.C:
                best = None
                for k in self.caches[i]:              # linear scan over all residents
                    if k in self.pinned[i]:
                        continue
                    key = (self._prim(i, k), k)
                    if best is None or key < best:
                        best = key
                k = best[1]
                e = self.caches[i].pop(k)
                dirty = e["cc"] > e["cs"]
                self.victims[i].append((k, dirty))
                if dirty:
                    pushes[i].append((k, e["p"], e["cc"]))
        for i in range(self.N):
            for k, p, cc in sorted(pushes[i], key=lambda x: x[0]):
                self._push(k, p, cc)

    def flush(self):
        for i in range(self.N):
            for k in sorted(self.caches[i]):
                e = self.caches[i][k]
                if e["cc"] > e["cs"]:
                    self._push(k, e["p"], e["cc"])
            self.caches[i] = {}
            self.pinned[i] = set()

    def global_row(self, k):
        return np.array(self._row(k), dtype=np.float32), self.cg.get(k, 0)
