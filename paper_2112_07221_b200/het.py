"""Thin ctypes binding of libhet.so (include/het.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of libhet.so.  The functions keep the C names; ``HetCache`` is a small
convenience wrapper over torch tensors.  There is no CPU fallback: if
libhet.so is missing this module raises on import of the library.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhet.so")

HET_LFU, HET_LRU, HET_LIGHT_LFU = 0, 1, 2
HET_S_INF = 0xFFFFFFFF
HET_CLOCK_AUTO = 0xFFFFFFFFFFFFFFFF
STATUS = {0: "HET_OK", 1: "HET_ERR_ARG", 2: "HET_ERR_KEY_RANGE", 3: "HET_ERR_PROTOCOL",
          4: "HET_ERR_CAPACITY", 5: "HET_ERR_OOM", 6: "HET_ERR_CUDA", 7: "HET_ERR_NCCL"}
HIT, EXP1, EXP2, MISS = 0, 1, 2, 3


class HetError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class het_dist_t(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p)]


class het_opts_t(ctypes.Structure):
    _fields_ = [("max_keys_per_call", ctypes.c_uint32), ("init_seed", ctypes.c_uint64),
                ("lfu_persist", ctypes.c_int), ("debug_log", ctypes.c_int),
                ("pin_threshold", ctypes.c_uint32), ("dense_max", ctypes.c_uint64)]


class het_stats_t(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in
                ["lookups", "keys", "unique", "hits", "exp1", "exp2", "misses", "evictions",
                 "dirty_pushes", "bytes_clock_tx", "bytes_clock_rx", "bytes_emb_tx", "bytes_emb_rx",
                 "launches"]] + [("resident", ctypes.c_uint32), ("capacity", ctypes.c_uint32),
                                 ("sticky_error", ctypes.c_int), ("pinned", ctypes.c_uint32)]

    def as_dict(self):
        return {f[0]: int(getattr(self, f[0])) for f in self._fields_}


EXPORTS = ["het_get_unique_id", "het_cache_create", "het_lookup", "het_update", "het_evict",
           "het_sync", "het_stats", "het_check", "het_read_global", "het_dense_allreduce",
           "het_debug_lookup_log", "het_debug_victims", "het_debug_dump_cache",
           "het_profile_enable", "het_profile_read", "het_cache_destroy", "het_last_error",
           "het_group_create", "het_group_lookup", "het_group_update", "het_group_evict",
           "het_group_sync", "het_group_dense_allreduce", "het_debug_eviction_plan", "het_prefetch"]

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, U32, U64, I, F, D = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int,
                            ctypes.c_float, ctypes.c_double)
    sig = {
        "het_get_unique_id": [P],
        "het_cache_create": [U64, U32, D, U32, I, P, P, P, P],
        "het_lookup": [P, P, U32, U64, P, P],
        "het_update": [P, P, U32, P, F, P],
        "het_evict": [P, P, U32, P],
        "het_sync": [P, P],
        "het_stats": [P, P],
        "het_check": [P],
        "het_read_global": [P, P, U32, P, P, P],
        "het_dense_allreduce": [P, P, U64, P],
        "het_debug_lookup_log": [P, P, P, P, P, P, P, P],
        "het_debug_victims": [P, P, P, U32, P, P],
        "het_debug_dump_cache": [P, P, P, P, P, P, P, U32, P, P],
        "het_profile_enable": [P, I],
        "het_profile_read": [P, P, P, P, U32, P],
        "het_cache_destroy": [P],
        "het_group_create": [U32, U64, U32, D, U32, I, P, P, P],
        "het_group_lookup": [P, U32, P, P, U64, P, P],
        "het_group_update": [P, U32, P, P, P, F, P],
        "het_group_evict": [P, U32, P, P, P],
        "het_group_sync": [P, U32, P],
        "het_group_dense_allreduce": [P, U32, P, U64, P],
        "het_debug_eviction_plan": [P, P, P],
        "het_prefetch": [P, P, U32, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.het_last_error.argtypes = [P]
    lib.het_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


_Tensor = None   # torch.Tensor once torch is imported (argument fast path)
_raw_stream = None   # torch's current raw CUDA stream of the current device


def _ptr(x):
    """Device or host address of a torch tensor / numpy array / int / None."""
    if _Tensor is not None and type(x) is _Tensor:   # the common case first (the e2e leg: per call)
        if not x.is_contiguous():
            raise ValueError("tensor arguments must be contiguous")
        return x.data_ptr()
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous()
        return x.data_ptr()
    raise TypeError(type(x))


def _stream(stream):
    global _Tensor, _raw_stream
    if stream is None:
        if _raw_stream is None:
            import torch
            if not torch.cuda.is_available():
                return None
            _Tensor = torch.Tensor
            get_raw, get_dev = getattr(torch._C, "_cuda_getCurrentRawStream", None), getattr(torch._C, "_cuda_getDevice", None)
            if get_raw is not None and get_dev is not None:
                _raw_stream = lambda: get_raw(get_dev())   # noqa: E731  (~10x cheaper than current_stream())
            else:
                _raw_stream = lambda: torch.cuda.current_stream().cuda_stream   # noqa: E731
        return _raw_stream()
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _check(h, rc, what):
    if rc != 0:
        msg = load().het_last_error(h).decode() if h else ""
        raise HetError(rc, f"{what}: {msg}")


# ----------------------------------------------------------------- C-named wrappers
def het_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(None, load().het_get_unique_id(buf), "het_get_unique_id")
    return buf.raw


def het_cache_create(rows, D, cache_frac, s, policy=HET_LFU, rank=0, world=1, unique_id=None,
                     max_keys_per_call=65536, init_seed=0, lfu_persist=1, stream=None, pin_threshold=0,
                     dense_max=0):
    lib = load()
    dist = None
    uid = None
    if world > 1:
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        dist = het_dist_t(rank, world, ctypes.cast(uid, ctypes.c_void_p))
    opts = het_opts_t(max_keys_per_call, init_seed, lfu_persist, 0, pin_threshold, dense_max)
    h = ctypes.c_void_p()
    rc = lib.het_cache_create(rows, D, cache_frac, s, policy,
                              ctypes.byref(dist) if dist is not None else None,
                              ctypes.byref(opts), _stream(stream), ctypes.byref(h))
    _check(None, rc, "het_cache_create")
    return h.value


def het_lookup(h, keys, n, clock, out, stream=None):
    _check(h, load().het_lookup(h, _ptr(keys), n, clock, _ptr(out), _stream(stream)), "het_lookup")


def het_prefetch(h, keys, n, stream=None):
    _check(h, load().het_prefetch(h, _ptr(keys), n, _stream(stream)), "het_prefetch")


def het_update(h, keys, n, grads, lr, stream=None):
    _check(h, load().het_update(h, _ptr(keys), n, _ptr(grads), ctypes.c_float(lr), _stream(stream)),
           "het_update")


def het_evict(h, keys, n, stream=None):
    _check(h, load().het_evict(h, _ptr(keys), n, _stream(stream)), "het_evict")


def het_sync(h, stream=None):
    _check(h, load().het_sync(h, _stream(stream)), "het_sync")


def het_check(h):
    _check(h, load().het_check(h), "het_check")


def het_stats(h) -> dict:
    st = het_stats_t()
    _check(h, load().het_stats(h, ctypes.byref(st)), "het_stats")
    return st.as_dict()


def het_read_global(h, keys, n, rows, cg, stream=None):
    _check(h, load().het_read_global(h, _ptr(keys), n, _ptr(rows), _ptr(cg), _stream(stream)),
           "het_read_global")


def het_dense_allreduce(h, buf, count, stream=None):
    _check(h, load().het_dense_allreduce(h, _ptr(buf), count, _stream(stream)), "het_dense_allreduce")


def het_profile_enable(h, on):
    _check(h, load().het_profile_enable(h, 1 if on else 0), "het_profile_enable")


def het_profile_read(h):
    cap = 64
    names = (ctypes.c_char * 32 * cap)()
    ms = (ctypes.c_double * cap)()
    cnt = (ctypes.c_uint64 * cap)()
    k = ctypes.c_uint32()
    _check(h, load().het_profile_read(h, names, ms, cnt, cap, ctypes.byref(k)), "het_profile_read")
    return {bytes(names[i]).split(b"\0")[0].decode(): (float(ms[i]), int(cnt[i])) for i in range(k.value)}


def _arr(ctype, xs):
    return (ctype * len(xs))(*xs)


def het_group_create(N, rows, D, cache_frac, s, policy=HET_LFU, max_keys_per_call=65536, init_seed=0,
                     lfu_persist=1, stream=None, pin_threshold=0, dense_max=0):
    """Loopback group: N workers on the current device (include/het.h); returns the N handles."""
    opts = het_opts_t(max_keys_per_call, init_seed, lfu_persist, 0, pin_threshold, dense_max)
    out = (ctypes.c_void_p * N)()
    _check(None, load().het_group_create(N, rows, D, cache_frac, s, policy, ctypes.byref(opts),
                                         _stream(stream), out), "het_group_create")
    return [out[i] for i in range(N)]


def het_group_lookup(hs, keys, n, clock, out, stream=None):
    N = len(hs)
    _check(hs[0], load().het_group_lookup(_arr(ctypes.c_void_p, hs), N, _arr(ctypes.c_void_p, [_ptr(k) for k in keys]),
                                          _arr(ctypes.c_uint32, n), clock,
                                          _arr(ctypes.c_void_p, [_ptr(o) for o in out]), _stream(stream)),
           "het_group_lookup")


def het_group_update(hs, keys, n, grads, lr, stream=None):
    N = len(hs)
    _check(hs[0], load().het_group_update(_arr(ctypes.c_void_p, hs), N, _arr(ctypes.c_void_p, [_ptr(k) for k in keys]),
                                          _arr(ctypes.c_uint32, n), _arr(ctypes.c_void_p, [_ptr(g) for g in grads]),
                                          ctypes.c_float(lr), _stream(stream)), "het_group_update")


def het_group_evict(hs, keys, n, stream=None):
    N = len(hs)
    k = None if keys is None else _arr(ctypes.c_void_p, [_ptr(x) for x in keys])
    nn = None if keys is None else _arr(ctypes.c_uint32, n)
    _check(hs[0], load().het_group_evict(_arr(ctypes.c_void_p, hs), N, k, nn, _stream(stream)), "het_group_evict")


def het_group_sync(hs, stream=None):
    _check(hs[0], load().het_group_sync(_arr(ctypes.c_void_p, hs), len(hs), _stream(stream)), "het_group_sync")


def het_group_dense_allreduce(hs, bufs, count, stream=None):
    _check(hs[0], load().het_group_dense_allreduce(_arr(ctypes.c_void_p, hs), len(hs),
                                                   _arr(ctypes.c_void_p, [_ptr(b) for b in bufs]), count,
                                                   _stream(stream)), "het_group_dense_allreduce")


def het_debug_eviction_plan(h):
    """The last update's eviction plan: mode, need, victims, T, K*, lowmask."""
    out = np.zeros(8, np.int64)
    _check(h, load().het_debug_eviction_plan(h, _ptr(out), _stream(None)), "het_debug_eviction_plan")
    return dict(zip(["mode", "need", "victims", "T", "Kstar", "lowmask"], [int(x) for x in out[:6]]))


def het_cache_destroy(h):
    if h:
        load().het_cache_destroy(h)


# ----------------------------------------------------------------- convenience wrapper
class HetCache:
    """One worker's cache (torch tensors in, torch tensors out)."""

    def __init__(self, rows, D, cache_frac, s, policy=HET_LFU, rank=0, world=1, unique_id=None,
                 max_keys_per_call=65536, init_seed=0, lfu_persist=1, pin_threshold=0, dense_max=0):
        import torch
        self.torch = torch
        self.rows, self.D, self.world, self.rank = rows, D, world, rank
        self.n_max = max_keys_per_call
        self.h = het_cache_create(rows, D, cache_frac, s, policy, rank, world, unique_id,
                                  max_keys_per_call, init_seed, lfu_persist, pin_threshold=pin_threshold,
                                  dense_max=dense_max)

    def close(self):
        if self.h:
            het_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup(self, keys, t, out=None):
        torch = self.torch
        n = keys.numel()
        if out is None:
            out = torch.empty((n, self.D), dtype=torch.float32, device=keys.device)
        het_lookup(self.h, keys, n, t, out)
        return out

    def update(self, keys, grads, lr):
        het_update(self.h, keys, keys.numel(), grads, lr)

    def prefetch(self, keys, stream=None):
        """NEXT-1: dedup of the next lookup's keys now (e.g. on a side stream)."""
        het_prefetch(self.h, keys, keys.numel(), stream)

    def step(self, keys, grads, out, lr, dense=None, side=None):
        """One training step of the sparse path: lookup (HET_CLOCK_AUTO) +
        update; with `dense` (N > 1) the dense all-reduce (Eq. 2) runs
        concurrently on the side stream (async communication)."""
        torch = self.torch
        n = keys.numel()
        cs = torch.cuda.current_stream()
        if dense is not None:
            side.wait_stream(cs)
            with torch.cuda.stream(side):
                het_dense_allreduce(self.h, dense, dense.numel(), stream=side)
        het_lookup(self.h, keys, n, HET_CLOCK_AUTO, out)
        het_update(self.h, keys, n, grads, lr)
        if dense is not None:
            cs.wait_stream(side)

    def capture_step(self, keys, grads, out, lr, dense=None):
        """Capture step() on static device buffers into a CUDA graph;
        replay() runs the whole step.  Run at least one uncaptured step first
        (lazy one-time attribute setup)."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream() if dense is not None else None
        with torch.cuda.graph(g, capture_error_mode="relaxed"):
            self.step(keys, grads, out, lr, dense, side)
        return g

    def evict(self, keys=None):
        if keys is None:
            het_evict(self.h, None, 0)
        else:
            het_evict(self.h, keys, keys.numel())

    def sync(self):
        het_sync(self.h)

    def stats(self):
        return het_stats(self.h)

    def read_global(self, keys):
        keys = np.ascontiguousarray(np.asarray(keys, np.int64))
        rows = np.zeros((keys.size, self.D), np.float32)
        cg = np.zeros(keys.size, np.uint32)
        het_read_global(self.h, keys, keys.size, rows, cg)
        return rows, cg

    def lookup_log(self):
        lib = load()
        n = self.n_max
        uniq = np.zeros(n, np.int64)
        inv = np.zeros(n, np.int32)
        perm = np.zeros(n, np.int32)
        seg = np.zeros(n + 1, np.int32)
        st = np.zeros(n, np.uint8)
        U = ctypes.c_uint32()
        _check(self.h, lib.het_debug_lookup_log(self.h, _ptr(uniq), _ptr(inv), _ptr(perm), _ptr(seg),
                                                _ptr(st), ctypes.byref(U), _stream(None)), "lookup_log")
        u = U.value
        return dict(unique=uniq[:u], inverse=inv, perm=perm, seg_off=seg[:u + 1], status=st[:u])

    def victims(self):
        lib = load()
        cap = 2 * self.n_max + 1
        k = np.zeros(cap, np.int64)
        d = np.zeros(cap, np.uint8)
        e = ctypes.c_uint32()
        _check(self.h, lib.het_debug_victims(self.h, _ptr(k), _ptr(d), cap, ctypes.byref(e),
                                             _stream(None)), "victims")
        return k[:e.value], d[:e.value]

    def dump_cache(self, cap=1 << 20, rows=True):
        return _dump_cache(self.h, self.D, rows)


class _Member:
    """Inspection view of one loopback worker (non-collective calls only)."""

    def __init__(self, h, D, n_max, rank, world):
        self.h, self.D, self.n_max, self.rank, self.world = h, D, n_max, rank, world

    stats = HetCache.stats
    read_global = HetCache.read_global
    lookup_log = HetCache.lookup_log
    victims = HetCache.victims

    def dump_cache(self, rows=True):
        return _dump_cache(self.h, self.D, rows)


class HetGroup:
    """N loopback workers on one GPU (het_group_*): every collective call takes
    per-worker lists and drives the workers phase by phase."""

    def __init__(self, N, rows, D, cache_frac, s, policy=HET_LFU, max_keys_per_call=65536, init_seed=0,
                 lfu_persist=1, pin_threshold=0, dense_max=0):
        import torch
        self.torch = torch
        self.N, self.rows, self.D, self.n_max = N, rows, D, max_keys_per_call
        self.hs = het_group_create(N, rows, D, cache_frac, s, policy, max_keys_per_call, init_seed, lfu_persist,
                                   pin_threshold=pin_threshold, dense_max=dense_max)
        self.workers = [_Member(h, D, max_keys_per_call, i, N) for i, h in enumerate(self.hs)]

    def close(self):
        if self.hs:
            for h in self.hs:
                het_cache_destroy(h)
            self.hs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup(self, keys, t):
        torch = self.torch
        outs = [torch.empty((k.numel(), self.D), dtype=torch.float32, device=k.device) for k in keys]
        het_group_lookup(self.hs, keys, [k.numel() for k in keys], t, outs)
        return outs

    def update(self, keys, grads, lr):
        het_group_update(self.hs, keys, [k.numel() for k in keys], grads, lr)

    def evict(self, keys=None):
        if keys is None:
            het_group_evict(self.hs, None, None)
        else:
            het_group_evict(self.hs, keys, [k.numel() for k in keys])

    def sync(self):
        het_group_sync(self.hs)

    def dense_allreduce(self, bufs):
        het_group_dense_allreduce(self.hs, bufs, bufs[0].numel())


def _dump_cache(h, D, rows=True):
    lib = load()
    m = ctypes.c_uint32()
    lib.het_debug_dump_cache(h, None, None, None, None, None, None, 0, ctypes.byref(m), _stream(None))  # size query
    mm = m.value
    keys = np.zeros(mm, np.int64)
    v = np.zeros((mm, D), np.float32) if rows else None
    p = np.zeros((mm, D), np.float32) if rows else None
    cs = np.zeros(mm, np.uint32)
    cc = np.zeros(mm, np.uint32)
    prim = np.zeros(mm, np.uint32)
    _check(h, lib.het_debug_dump_cache(h, _ptr(keys), _ptr(v), _ptr(p), _ptr(cs), _ptr(cc),
                                       _ptr(prim), mm, ctypes.byref(m), _stream(None)), "dump")
    return dict(keys=keys, v=v, p=p, cs=cs, cc=cc, prim=prim)
