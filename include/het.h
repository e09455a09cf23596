/*
 * het.h — C-ABI of the B200-native HET cached-embedding hot path.
 *
 * HET (Miao et al., "HET: Scaling out Huge Embedding Model Training via
 * Cache-enabled Distributed Framework", arXiv 2112.07221, PVLDB).  Citations
 * "P:n" are lines of /root/reference/PAPER.md (canonical copy 168-810);
 * "Rn" are the readings of the paper listed in DESIGN.md.
 *
 * One handle = one worker (one GPU, one process).  The worker owns a cache
 * embedding table in HBM and, with N workers, the 1/N hash shard
 * of the global embedding table and its global clocks (R15:
 * owner(k) = k mod N, local row = k div N).
 *
 * Pointers: every `keys`, `grads`, `out`, `rows`, `cg` argument may be a
 * device pointer (cudaMalloc / torch CUDA tensor) or a host pointer (pinned
 * or pageable); host buffers are staged through library-owned device
 * buffers with cudaMemcpyAsync on `stream`.  The caller owns its buffers and
 * keeps them alive until `stream` has completed the call.  Layouts: keys
 * int64[n]; rows float32[n][D] row-major; clocks uint32[n].
 *
 * Streams: all device work is enqueued on `stream` (a cudaStream_t); calls
 * return without host synchronisation except het_sync, het_stats, the debug
 * exports and (N > 1) the count exchanges of the all-to-alls.  One exception
 * in where, not when: het_update with host gradients right after a
 * het_lookup with host rows out (N = 1) runs its kernels on a library stream
 * that waits for the lookup's kernels only (so they overlap the rows' D2H),
 * and `stream` waits for them: the call still completes on `stream`.
 *
 * Errors: argument/shape/protocol errors are returned synchronously and leave
 * the cache untouched.  Errors detected on the device (a key outside
 * [0, rows), cache entries exhausted) abort the rest of that call on the
 * device, are latched ("sticky"), and are returned by the next het_sync /
 * het_stats / het_check.
 *
 * Collectives: with N > 1, het_lookup, het_update, het_evict, het_sync,
 * het_read_global and het_dense_allreduce are collective — every rank calls
 * them in the same order with the same clock (n may differ, including 0).
 *
 * Loopback group (het_group_*): N workers in ONE process on ONE device, with
 * the same per-worker state, kernels and peer-memory exchange records as N
 * processes on N GPUs, but the inboxes are plain device allocations shared by
 * pointer (no CUDA IPC, no NCCL) and each collective call is driven phase by
 * phase over the members -- phase k of every worker before phase k+1 of any --
 * so no kernel ever waits for a flag another kernel has not yet set.  Used to
 * test the N-worker protocol (CheckValid condition (2), owner-side sync/fetch,
 * carried eviction pushes, Eq. 2) on a single GPU.
 */
#ifndef HET_H
#define HET_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct het_cache* het_cache_t;     /* opaque; the library owns all table/cache/hash/comm state */
typedef struct CUstream_st* het_stream_t;  /* == cudaStream_t */

/* HET_LIGHT_LFU ("a light-weighted version of LFU"): an entry whose LFU
 * count reaches opts.pin_threshold (default 64) gets a direct
 * access index -- pinned: no more count maintenance, never an overflow victim
 * (S:275); never demoted.  Promotions go in ascending key order while
 * fewer than floor(C/2) entries are pinned (reading R27). */
typedef enum { HET_LFU = 0, HET_LRU = 1, HET_LIGHT_LFU = 2 } het_policy_t;

typedef enum {
  HET_OK = 0,
  HET_ERR_ARG = 1,        /* bad argument or shape */
  HET_ERR_KEY_RANGE = 2,  /* a key outside [0, rows) (sticky) */
  HET_ERR_PROTOCOL = 3,   /* write without matching read */
  HET_ERR_CAPACITY = 4,   /* cache entries or per-call capacity exhausted */
  HET_ERR_OOM = 5,
  HET_ERR_CUDA = 6,
  HET_ERR_NCCL = 7
} het_status_t;

#define HET_S_INF 0xFFFFFFFFu  /* s = infinity: no clock checks, every hit valid (R4) */
/* clock_t value asking the library for its own device-side iteration counter
 * (0, 1, 2, ... per lookup): lets a captured CUDA graph of a step be replayed. */
#define HET_CLOCK_AUTO 0xFFFFFFFFFFFFFFFFull

typedef struct {
  int rank;                    /* this worker, 0 <= rank < world */
  int world;                   /* N workers = GPUs */
  const void* nccl_unique_id;  /* 128-byte ncclUniqueId from het_get_unique_id on rank 0 */
} het_dist_t;

typedef struct {
  uint32_t max_keys_per_call;  /* n_max: bound on n for lookup/update/evict (sizes all scratch) */
  uint64_t init_seed;          /* seed of the initial table W0 (R14); 0 = default 2112072210 */
  int lfu_persist;             /* 1 (default): LFU counts persist across evictions (R7); 0: reset */
  int debug_log;               /* reserved */
  uint32_t pin_threshold;      /* HET_LIGHT_LFU promotion count; 0 = default 64 */
  uint64_t dense_max;          /* N > 1: floats of the peer-memory dense all-reduce staging, set up at
                                  create (0 = default 2^22); larger het_dense_allreduce calls take NCCL */
} het_opts_t;

typedef struct {
  uint64_t lookups, keys, unique, hits, exp1, exp2, misses, evictions, dirty_pushes;
  uint64_t bytes_clock_tx, bytes_clock_rx, bytes_emb_tx, bytes_emb_rx;  /* wire bytes (N > 1) */
  uint64_t launches;           /* kernels launched by the library so far */
  uint32_t resident, capacity; /* |cache| and C */
  int sticky_error;            /* het_status_t latched on the device, 0 = none */
  uint32_t pinned;             /* HET_LIGHT_LFU: pinned (direct-access) entries */
} het_stats_t;

/* ncclUniqueId (128 bytes) for multi-GPU bootstrap; call on rank 0, broadcast. */
het_status_t het_get_unique_id(void* out128);

/* Create one worker ("core methods of the HET client library").
 *   rows       R, keys are int64 in [0, R) (R15); R <= 2^32
 *   D          embedding dimension, multiple of 4
 *   cache_frac C = floor(cache_frac * R) cache entries per worker (R10); 0 = no cache
 *   s          staleness threshold, HET_S_INF = infinity
 *   policy     LFU, LRU or light-LFU eviction
 *   dist       NULL for a single worker, else rank/world/ncclUniqueId
 *   opt        NULL for defaults (n_max = 65536)
 * Allocates everything up front (no allocation on the hot path) and writes
 * W0 (R14) with c_g = 0.  Synchronises `stream` before returning. */
het_status_t het_cache_create(uint64_t rows, uint32_t D, double cache_frac, uint32_t s,
                              het_policy_t policy, const het_dist_t* dist, const het_opts_t* opt,
                              het_stream_t stream, het_cache_t* out);

/* Het.Read (Alg. 2) of one mini-batch: dedup,
 * Cache.Find, CheckValid, Evict(k)+Fetch(k) of expired hits
 * fused into one sync (R5), Fetch of misses,
 * LFU/LRU touch, then Cache.Get: out[pos] = cached row of keys[pos]
 * (lookup semantics P:349-355).  clock_t = the caller's iteration t,
 * strictly increasing (LRU tick, R8), or HET_CLOCK_AUTO.  out: float32[n][D].
 * Capturable into a CUDA graph (device pointers, HET_CLOCK_AUTO, N = 1). */
het_status_t het_lookup(het_cache_t h, const int64_t* keys, uint32_t n, uint64_t clock_t,
                        float* out, het_stream_t stream);

/* Message fusion's prefetch (NEXT-1; "pre-fetch the next mini-batch
 * of data in advance"): run the dedup of the NEXT het_lookup's keys now -- for
 * example on a side stream while the dense backward and het_update of this
 * step run.  The next het_lookup with the same `keys` pointer and `n` skips its
 * own dedup; any other next lookup ignores the prefetch.  The dedup is a
 * function of the keys alone, so every result is unchanged; a key outside
 * [0, rows) is reported by that lookup (sticky HET_ERR_KEY_RANGE).  The
 * caller orders the lookup after the prefetch (same stream or an event) and
 * keeps `keys` unchanged in between.  A no-op on paths without a separate
 * dedup kernel (n > 16384, HET_NO_FUSED).  Local: allowed on loopback
 * members and at N > 1 without the other ranks. */
het_status_t het_prefetch(het_cache_t h, const int64_t* keys, uint32_t n, het_stream_t stream);

/* Het.Write (Alg. 3) for the keys of the immediately preceding
 * het_lookup (a write of keys the read did not return is a
 * protocol violation).  n != the lookup's n: HET_ERR_PROTOCOL, returned at
 * once.  `keys` is the lookup's pointer: accepted as is (the library reads it
 * no further).  Any other buffer is compared on the device with the lookup's
 * dedup, position by position; a mismatch latches HET_ERR_PROTOCOL (sticky,
 * reported by het_check / het_sync) and the update is skipped entirely (no
 * partial mutation).  The lookup's dedup is reused: per unique key
 * acc = sum of grads[pos] in ascending position (R11), delta = -lr * acc,
 * v += delta, pending += delta, c_c += 1; then the
 * overflow Evict() (R9).  grads: float32[n][D]. */
het_status_t het_update(het_cache_t h, const int64_t* keys, uint32_t n, const float* grads,
                        float lr, het_stream_t stream);

/* Het.Cache.Evict: keys != NULL evicts those keys (pushing
 * accumulated deltas and c_c to their owner, c_g = max(c_g, c_c)); keys ==
 * NULL runs the overflow eviction down to C entries. */
het_status_t het_evict(het_cache_t h, const int64_t* keys, uint32_t n, het_stream_t stream);

/* End-of-run flush (R16): push every dirty entry, empty the cache,
 * synchronise `stream`, return any sticky device error. */
het_status_t het_sync(het_cache_t h, het_stream_t stream);

/* Counters since create (synchronises the device). */
het_status_t het_stats(het_cache_t h, het_stats_t* out);

/* Return the sticky device error without other side effects (synchronises). */
het_status_t het_check(het_cache_t h);

/* Read global rows W[k] and clocks c_g[k] (inspection/tests).  With N > 1
 * only keys owned by this rank (k mod N == rank) may be passed. */
het_status_t het_read_global(het_cache_t h, const int64_t* keys, uint32_t n, float* rows,
                             uint32_t* cg, het_stream_t stream);

/* Eq. 2 dense synchronisation: buf[0..count) <- mean over the N
 * workers (NCCL all-reduce sum, then scale by 1/N); identity at N = 1. */
het_status_t het_dense_allreduce(het_cache_t h, float* buf, uint64_t count, het_stream_t stream);

/* Debug / parity exports of the last call (synchronise `stream`; host or
 * device destinations).  Unique keys ascending, inverse/perm int32[n],
 * seg_off int32[U+1], status uint8[U] (0 HIT, 1 EXP1, 2 EXP2, 3 MISS). */
het_status_t het_debug_lookup_log(het_cache_t h, int64_t* uniq, int32_t* inverse, int32_t* perm,
                                  int32_t* seg_off, uint8_t* status, uint32_t* U,
                                  het_stream_t stream);
/* Victims of the last overflow eviction, ascending key, with dirty flags. */
het_status_t het_debug_victims(het_cache_t h, int64_t* keys, uint8_t* dirty, uint32_t cap,
                               uint32_t* e, het_stream_t stream);
/* Resident entries ascending by key: v/p float32[m][D], clocks, policy primary
 * (LFU count or LRU tick).  cap bounds m; NULL arrays are skipped. */
het_status_t het_debug_dump_cache(het_cache_t h, int64_t* keys, float* v, float* p, uint32_t* cs,
                                  uint32_t* cc, uint32_t* prim, uint32_t cap, uint32_t* m,
                                  het_stream_t stream);

/* The last update's overflow-eviction plan (R9),
 * for inspection: out8 = {mode (0 none, 1 LFU count bitmaps, 2 generic
 * selection), need = |cache| - C, victims, threshold T (count or tick), the
 * largest victim key among primary T (mode 1), counts below T present
 * (bitmask, mode 1), 0, 0}.  Synchronises `stream`. */
het_status_t het_debug_eviction_plan(het_cache_t h, int64_t* out8, het_stream_t stream);

/* Per-kernel timing with CUDA events on the launching stream (bench). */
het_status_t het_profile_enable(het_cache_t h, int on);
/* Fills up to cap (name, total ms, launches) records; returns count in *k. */
het_status_t het_profile_read(het_cache_t h, char (*names)[32], double* ms, uint64_t* launches,
                              uint32_t cap, uint32_t* k);

/* ---- loopback group (see "Loopback group" above) ----
 * het_group_create: N (2..16) workers rank 0..N-1 on the current device, all
 * with the given arguments; out[N] receives the handles in rank order.  The
 * handles are used with het_group_* (every member, rank order, in `hs`) and
 * with the non-collective calls (het_stats, het_check, het_read_global of
 * owned keys, het_debug_*); het_lookup / het_update / het_evict / het_sync /
 * het_dense_allreduce on a member return HET_ERR_PROTOCOL.  Destroy every
 * member with het_cache_destroy.  keys[i], n[i], out[i], grads[i], bufs[i]
 * are worker i's arguments of the corresponding single-worker call. */
het_status_t het_group_create(uint32_t N, uint64_t rows, uint32_t D, double cache_frac, uint32_t s,
                              het_policy_t policy, const het_opts_t* opt, het_stream_t stream,
                              het_cache_t* out);
/* Alg. 2 for every worker: dedup; probe + request build; owner
 * link; owner process (U4 of the previous update, CheckValid condition (2)
 * P:448, sync pushes P:442-443, responses P:439); install + Get. */
het_status_t het_group_lookup(const het_cache_t* hs, uint32_t N, const int64_t* const* keys,
                              const uint32_t* n, uint64_t clock_t, float* const* out,
                              het_stream_t stream);
/* Alg. 3 for every worker; eviction pushes go to the owners'
 * inboxes and are applied by the next round (U4 precedes the next L3). */
het_status_t het_group_update(const het_cache_t* hs, uint32_t N, const int64_t* const* keys,
                              const uint32_t* n, const float* const* grads, float lr,
                              het_stream_t stream);
/* Cache.Evict for every worker; keys == NULL: overflow Evict(). */
het_status_t het_group_evict(const het_cache_t* hs, uint32_t N, const int64_t* const* keys,
                             const uint32_t* n, het_stream_t stream);
/* End-of-run flush (R16) of every worker; synchronises `stream`. */
het_status_t het_group_sync(const het_cache_t* hs, uint32_t N, het_stream_t stream);
/* Eq. 2: bufs[i][0..count) <- mean over the workers, bitwise equal
 * on every worker; count must fit the staging (opts.dense_max). */
het_status_t het_group_dense_allreduce(const het_cache_t* hs, uint32_t N, float* const* bufs,
                                       uint64_t count, het_stream_t stream);

het_status_t het_cache_destroy(het_cache_t h);
const char* het_last_error(het_cache_t h);

#ifdef __cplusplus
}
#endif
#endif /* HET_H */
