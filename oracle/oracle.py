"""ctypes wrapper of the C++ HET cache-protocol oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  It shares nothing with the
CUDA path (paper_2112_07221_b200/); see het_oracle.cpp for the protocol steps
and their PAPER.md citations.

Parity pins: every function here is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py (SPEC worked examples, the paper's closed rules, closed
forms for N=1, and bit-exact agreement with the independent brute-force
implementation tests/brute.py).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "het_oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")

S_INF = 0xFFFFFFFF
LFU, LRU, LIGHT_LFU = 0, 1, 2
PIN_DEFAULT = 64        # light-LFU promotion threshold (R27)
PINNED = 0xFFFFFFFE     # dump_cache()["tick"] of a pinned (direct-access) entry
HIT, EXP1, EXP2, MISS = 0, 1, 2, 3
INIT_SEED = 2112072210
STAT_NAMES = ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses",
              "evictions", "dirty_pushes"]


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O2 -ffp-contract=off: fp32, no FMA, R17)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared",
               "-fPIC", "-o", LIB, SRC]
        subprocess.check_call(cmd)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P, I64, U32, U64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        lib.orc_create.restype = P
        lib.orc_create.argtypes = [I64, U32, I64, U32, I, I, I, U64, I64, U32]
        lib.orc_destroy.argtypes = [P]
        lib.orc_lookup.restype = I
        lib.orc_lookup.argtypes = [P, U64, P, P, P]
        lib.orc_update.restype = I
        lib.orc_update.argtypes = [P, P, ctypes.c_float]
        lib.orc_flush.restype = I
        lib.orc_flush.argtypes = [P]
        lib.orc_evict_keys.restype = I
        lib.orc_evict_keys.argtypes = [P, P, P]
        lib.orc_evict_overflow.restype = I
        lib.orc_evict_overflow.argtypes = [P]
        lib.orc_num_unique.restype = I64
        lib.orc_num_unique.argtypes = [P, I]
        lib.orc_get_lookup_log.argtypes = [P, I, P, P, P, P, P]
        lib.orc_num_victims.restype = I64
        lib.orc_num_victims.argtypes = [P, I]
        lib.orc_get_victims.argtypes = [P, I, P, P]
        lib.orc_get_stats.argtypes = [P, I, P]
        lib.orc_cache_size.restype = I64
        lib.orc_cache_size.argtypes = [P, I]
        lib.orc_dump_cache.argtypes = [P, I, P, P, P, P, P, P, P]
        lib.orc_read_global.argtypes = [P, P, I64, P, P]
        lib.orc_set_track_div.argtypes = [P, I64]
        lib.orc_w0.restype = ctypes.c_float
        lib.orc_w0.argtypes = [U64, I64, U32]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def capacity(cache_frac: float, R: int) -> int:
    """C = floor(cache_frac * R) entries per worker (R10)."""
    return int(math.floor(cache_frac * float(R)))


class Oracle:
    """N lock-step workers + the global table (one logical server)."""

    def __init__(self, R: int, D: int, C: int, s: int, policy: int = LFU, N: int = 1,
                 lfu_persist: int = 1, seed0: int = INIT_SEED, track_div: int = 1,
                 pin_threshold: int = PIN_DEFAULT):
        """policy: LFU, LRU or LIGHT_LFU (an entry whose count reaches
        `pin_threshold` gets a direct access index -- pinned, no more count
        maintenance, exempt from eviction; at most floor(C/2) pinned, R27)."""
        self.lib = _load()
        self.R, self.D, self.C, self.s, self.policy, self.N = R, D, C, s, policy, N
        self.h = self.lib.orc_create(R, D, C, s, policy, N, lfu_persist, seed0, track_div,
                                     pin_threshold if policy == LIGHT_LFU else 0)
        self._n = [0] * N

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.orc_destroy(h)
            self.h = None

    @staticmethod
    def _cat(keys_list):
        keys = [np.ascontiguousarray(np.asarray(k, dtype=np.int64)).reshape(-1) for k in keys_list]
        n_per = np.array([k.size for k in keys], dtype=np.int64)
        cat = np.concatenate(keys) if keys else np.zeros(0, np.int64)
        return np.ascontiguousarray(cat), n_per

    def lookup(self, t: int, keys_list, want_out: bool = True):
        """Het.Read for every worker (Alg. 2); returns per-worker out rows [n_i, D]."""
        assert len(keys_list) == self.N
        cat, n_per = self._cat(keys_list)
        out = np.zeros((cat.size, self.D), np.float32) if (want_out and self.D) else None
        rc = self.lib.orc_lookup(self.h, t, _ptr(cat), _ptr(n_per), _ptr(out))
        if rc:
            raise ValueError(f"oracle lookup error {rc}")
        self._n = list(n_per)
        if out is None:
            return None
        res, b = [], 0
        for n in self._n:
            res.append(out[b:b + n])
            b += n
        return res

    def update(self, grads_list, lr: float):
        """Het.Write for every worker (Alg. 3), including the overflow Evict()."""
        g = None
        if grads_list is not None and self.D:
            g = np.ascontiguousarray(np.concatenate(
                [np.asarray(x, np.float32).reshape(-1, self.D) for x in grads_list]))
        rc = self.lib.orc_update(self.h, _ptr(g), ctypes.c_float(lr))
        if rc:
            raise ValueError(f"oracle update error {rc}")

    def flush(self):
        self.lib.orc_flush(self.h)

    def evict_keys(self, keys_list):
        cat, n_per = self._cat(keys_list)
        self.lib.orc_evict_keys(self.h, _ptr(cat), _ptr(n_per))

    def evict_overflow(self):
        self.lib.orc_evict_overflow(self.h)

    def lookup_log(self, i: int):
        U = self.lib.orc_num_unique(self.h, i)
        n = self._n[i]
        d = dict(unique=np.zeros(U, np.int64), inverse=np.zeros(n, np.int32),
                 perm=np.zeros(n, np.int32), seg_off=np.zeros(U + 1, np.int32),
                 status=np.zeros(U, np.uint8))
        self.lib.orc_get_lookup_log(self.h, i, _ptr(d["unique"]), _ptr(d["inverse"]),
                                    _ptr(d["perm"]), _ptr(d["seg_off"]), _ptr(d["status"]))
        return d

    def victims(self, i: int):
        e = self.lib.orc_num_victims(self.h, i)
        k = np.zeros(e, np.int64)
        dirty = np.zeros(e, np.uint8)
        self.lib.orc_get_victims(self.h, i, _ptr(k), _ptr(dirty))
        return k, dirty

    def stats(self, i: int):
        a = np.zeros(9, np.uint64)
        self.lib.orc_get_stats(self.h, i, _ptr(a))
        return {k: int(v) for k, v in zip(STAT_NAMES, a)}

    def cache_size(self, i: int) -> int:
        return int(self.lib.orc_cache_size(self.h, i))

    def dump_cache(self, i: int):
        m = self.cache_size(i)
        D = self.D
        d = dict(keys=np.zeros(m, np.int64), v=np.zeros((m, D), np.float32),
                 p=np.zeros((m, D), np.float32), cs=np.zeros(m, np.uint32),
                 cc=np.zeros(m, np.uint32), count=np.zeros(m, np.uint32),
                 tick=np.zeros(m, np.uint32))
        self.lib.orc_dump_cache(self.h, i, _ptr(d["keys"]), _ptr(d["v"]) if D else None,
                                _ptr(d["p"]) if D else None, _ptr(d["cs"]), _ptr(d["cc"]),
                                _ptr(d["count"]), _ptr(d["tick"]))
        return d

    def set_track_div(self, track_div: int):
        """Bench only: which keys carry row values from now on (a clocks-only
        fill, then full rows).  Entries gaining rows get the server row as at
        a Fetch, so row values after the switch are not the protocol's."""
        self.lib.orc_set_track_div(self.h, int(track_div))

    def read_global(self, keys):
        keys = np.ascontiguousarray(np.asarray(keys, np.int64).reshape(-1))
        rows = np.zeros((keys.size, self.D), np.float32) if self.D else None
        cg = np.zeros(keys.size, np.uint32)
        self.lib.orc_read_global(self.h, _ptr(keys), keys.size, _ptr(rows), _ptr(cg))
        return rows, cg


def w0(key: int, d: int, seed0: int = INIT_SEED) -> float:
    return float(_load().orc_w0(seed0, key, d))
