// Internal state and device helpers of libhet (not part of the C-ABI).
//
// Layout in HBM (per rank = per worker):
//   server shard (R15 owner = k mod N, local row = k div N)
//     W   float[rows_local][D]          global embedding rows this rank owns
//     cg  u32[rows_local]               global Lamport clocks c_g
//   worker cache, struct-of-arrays over Ecap = C + 2*n_max entries
//     ekey i64[Ecap] (-1 = free)  v,p float[Ecap][D]  cs,cc u32[Ecap]
//     eprim u32[Ecap]  (LFU count or LRU tick: the policy's primary order key)
//     fstack i32[Ecap] + ctl.ftop       free-entry stack
//   open-addressing hash (Cache.Find): hslot u64[S] = key << 32 | entry
//     (keys < 2^32, R15), S = pow2 >= 4*Ecap, 32-slot aligned windows probed
//     by one warp: one 256 B load returns the entry with the match
//   count_by_key u32[R]                 persistent LFU counts (R7)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <cassert>

namespace het {

// Bounds-checked builds (HET_DIAG=HET_BOUNDS): device asserts on the indices
// the hot kernels compute -- free-stack slots, entries, inbox slots, sort
// positions (compute-sanitizer is not available on the GPU pool).
#ifdef HET_BOUNDS
#define HET_ASSERT(c) assert(c)
#else
#define HET_ASSERT(c) do {} while (0)
#endif

constexpr uint32_t S_INF = 0xFFFFFFFFu;
// hash slot word: key << 32 | entry (entry >= 0); EMPTY ends a probe, TOMB does not
constexpr uint64_t HS_EMPTY = ~0ull;                  // entry field -1
constexpr uint64_t HS_TOMB = 0xFFFFFFFFFFFFFFFEull;   // entry field -2
__host__ __device__ __forceinline__ uint64_t hs_pack(int64_t key, int32_t e) {
  return ((uint64_t)key << 32) | (uint32_t)e;
}
__device__ __forceinline__ bool hs_is(uint64_t w, int64_t key) {   // a live slot of `key`
  return (w >> 32) == (uint64_t)key && (int32_t)(uint32_t)w >= 0;
}
__device__ __forceinline__ int32_t hs_val(uint64_t w) { return (int32_t)(uint32_t)w; }
constexpr uint32_t EP_FREE = 0xFFFFFFFFu;  // eprim of a free entry
constexpr uint32_t EP_PIN = 0xFFFFFFFEu;   // eprim of a light-LFU pinned entry (R27): never a victim
constexpr int LFU_CB_MAX = 16;             // LFU count values kept in key bitmaps
constexpr int LFU_BLK_SHIFT = 12;          // 4096 keys per bitmap block counter

enum : uint8_t { ST_HIT = 0, ST_EXP1 = 1, ST_EXP2 = 2, ST_MISS = 3, ST_NEEDQ = 4,
                 ST_SKIP = 5 /* rmode: not a key's first sorted position */ };

// device counters (u64), order shared with het_stats_t
enum {
  C_UNIQUE = 0, C_HITS, C_EXP1, C_EXP2, C_MISSES, C_EVICTIONS, C_DIRTY_PUSHES, C_LOOKUPS, C_KEYS,
  C_BCLK_TX, C_BCLK_RX, C_BEMB_TX, C_BEMB_RX, C_NUM
};
constexpr uint64_t CLOCK_AUTO = ~0ull;   // HET_CLOCK_AUTO: device-side iteration counter

// small control block in device memory
struct Ctl {
  int32_t U;            // unique keys of the current call
  int32_t ftop;         // free-stack top (number of free entries)
  int32_t n_tomb;       // tombstones in the hash table
  int32_t abort;        // current call aborted (sticky error raised)
  int32_t err;          // sticky error code (het_status_t), 0 = none
  int32_t rebuild;      // hash rebuild requested for this step
  // eviction selection state (K8)
  int64_t need;         // |cache| - C
  uint32_t base;        // lower bound of all residents' primaries
  uint32_t T;           // threshold primary
  int64_t needT;        // victims still needed among prim == T
  int32_t nvict;        // victims emitted
  int32_t ncand;        // candidates with prim == T
  int32_t nsub;         // sub-candidates in key bucket kb1
  uint32_t kb1;         // key bucket (top bits) of the boundary
  int64_t need2;        // victims still needed among sub-candidates
  uint32_t T_last;      // previous eviction threshold (valid lower bound)
  uint32_t min_install; // min primary among this step's installs
  int32_t resolved;     // selection resolved (0/1)
  int32_t generic;      // run the generic (scan) selection this step
  int32_t vmode;        // victims list holds 0 = entry indices, 1 = keys
  int32_t pad3_;
  int32_t dd_done;      // blocks finished in the fused dedup (last-block pattern)
  int32_t lk_done;      // blocks finished in the fused lookup (light-LFU: the last one applies the promotions)
  int32_t emode;        // eviction this step: 0 none, 1 LFU bitmap threshold, 2 generic
  int32_t rebuild_req;  // hash rebuild requested for the next update
  uint32_t lk_seq;      // lookup sequence number
  int32_t nsel;         // victim keys extracted by the fused update
  uint32_t plan_seq;    // fused update: plan of round lk_seq published
  int32_t ntask;        // fused update: non-empty bitmap blocks to extract
  int32_t ext_next;     // work queue cursors
  int32_t ext_done;
  int32_t find_next;
  int32_t pad6_;
  uint32_t lowmask;     // bit c set: some resident has LFU count c < T (snapshot for enumeration)
  int64_t Kstar;        // LFU bitmap path: largest victim key among count == T
  uint64_t t_cur;       // clock of the current call (LRU tick)
  uint64_t t_auto;      // next automatic clock (HET_CLOCK_AUTO)
  // multi-GPU exchange bookkeeping
  int32_t nq;           // clock queries built this call
  int32_t nreq;         // sync/fetch requests built this call
  int32_t npush;        // eviction pushes built this call
  int32_t pad2_;
  // segment reduce (large batches): heavy keys per size bucket floor(log2(count))
  int32_t nbucket[32];
  // light-LFU (R27): promotion candidates of the current lookup, pinned entries
  int32_t npin_cand;
  int32_t pad7_;
  int64_t npinned;
  // deferred overflow eviction (fused path, LFU bitmap plan): the update lists
  // the victims of Evict(), the first kernel of the next call
  // evicts them before anything reads or changes the cache
  int32_t ev_pending;   // vsel[0, ev_nsel) still to evict
  int32_t ev_nsel;
  int32_t ev_ftop0;     // free-stack top when they were listed: victim i frees into fstack[ev_ftop0 + i]
  int32_t ext_blocks;   // extraction blocks finished (last-block counter)
  uint32_t plan_flag;   // lk_seq of the published plan (update: block 0 -> the other blocks)
  int32_t ev_done;      // eviction blocks finished (last-block counter)
};

struct Dev {
  // config
  int64_t R; uint32_t D; int64_t C; uint32_t s; int policy; int lfu_persist;
  int rank, world; uint64_t seed0; int kbits;  // bits of R-1
  // server shard
  float* W; uint32_t* cg; int64_t rows_local;
  // cache entries
  int64_t Ecap; int64_t* ekey; float* v; float* p; uint32_t* cs; uint32_t* cc;
  uint32_t* eprim; int32_t* fstack;
  uint32_t* estep;   // lookup sequence number that last touched the entry
  // hash
  uint64_t* hslot; int hbits; uint64_t hmask;
  uint32_t* count_by_key;
  Ctl* ctl; unsigned long long* cnt;
  // LFU count bitmaps (P:632 LFU): bit (c, key) set iff
  // key is resident with count c < lfu_cb; bcnt = set bits per 4096-key block
  int lfu_cb; int64_t bm_words; int64_t nbk; int64_t nbk2;
  uint32_t* bm; uint32_t* bcnt; uint32_t* bcnt2; int32_t* pop;   // bcnt2: per 64 blocks
  // light-LFU (R27): promotion threshold (0 = off), cap floor(C/2),
  // candidates (key, entry) of the current lookup, applied by k_pin_apply
  uint32_t pin_thr; int64_t pin_max; int64_t* pin_k; int32_t* pin_e;
};

// light-LFU touch (lane 0 of the key's warp): an entry that just reached the
// threshold becomes a promotion candidate; k_pin_apply pins the candidates in
// ascending key order while fewer than pin_max entries are pinned
__device__ __forceinline__ void unpin_count(const Dev& s, uint32_t prim) {   // a pinned entry leaves the cache
  if (prim == EP_PIN) atomicAdd(reinterpret_cast<unsigned long long*>(&s.ctl->npinned), ~0ull);
}
__device__ __forceinline__ void pin_candidate(const Dev& s, int64_t key, int32_t e, uint32_t newc) {
  if (s.pin_thr && newc >= s.pin_thr && newc != EP_PIN && newc != EP_FREE) {
    const int i = atomicAdd(&s.ctl->npin_cand, 1);
    s.pin_k[i] = key;
    s.pin_e[i] = e;
  }
}

// Per-call scratch (sized by n_max at create)
//
// Indexing of the per-key arrays (status, uentry, urec, upos, inverse):
//   rmode 0: by unique index u in [0, U) (compact dedup: uniq, seg_off)
//   rmode 1: by sorted position r in [0, n) of the key's first occurrence
//            (N = 1 fused path): the dedup leaves the sorted composites in
//            sortbuf0 and perm, with no compaction pass; a key's segment is
//            [r, next key change); non-head positions carry urec[r].x = -1.
//            het_debug_lookup_log compacts on demand (k_compact_log).
struct Call {
  int n;                       // occurrences in this call
  int rmode;                   // 1: per-key arrays indexed by sorted position (see above)
  int pbits;                   // position bits of the sort composites (key << pbits | pos)
  uint64_t t;                  // caller clock (LRU tick)
  const int64_t* keys;         // [n] device
  int64_t* uniq;               // [n_max]
  int32_t* inverse;            // [n_max]
  int32_t* perm;               // [n_max]
  int32_t* seg_off;            // [n_max+1]
  uint8_t* status;             // [n_max]
  int32_t* uentry;             // [n_max] entry index per unique key
  uint64_t* sortbuf0;          // [n_max] composite sort buffers (large path)
  uint64_t* sortbuf1;
  int32_t* blockbuf;           // block counts for scans
  int32_t* hlist;              // [n_max] heavy keys of the current update (segment reduce)
  int4* urec;                  // [n_max] per unique key, lookup -> update: {entry, j0, cnt | dirty << 31, c_c}
  int4* upos;                  // [n_max] its first four batch positions (ascending)
  int32_t* ucnt;               // [n_max] rmode at N > 1: the key's occurrences (uniq[r] holds the key)
  int32_t* pref_bad;           // het_prefetch: 1 when the prefetched keys held one outside [0, R)
  uint64_t* ucslot;            // [n_max] N > 1: a miss's hash insert slot from the probe (warp_find_cand)
  uint64_t* ucword;            // [n_max]         and that slot's word
  uint8_t* dbg_status;         // [n_max] rmode: compacted status (debug export)
  int32_t* dbg_inverse;        // [n_max] rmode: compacted inverse (debug export)
  int32_t* dbg_U;              // rmode: unique keys of the compacted log
  float* hbuf;                 // [ceil(D/16)][n_max][16] heavy keys' gradient rows, key-contiguous, slice-major
  int hcap;                    // n_max (rows per hbuf slice plane)
};

__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27; x *= 0x94D049BB133111EBull;
  x ^= x >> 31; return x;
}

// R14 initial row value (the CUDA side's own copy of the counter hash)
__device__ __forceinline__ float init_w0(uint64_t seed0, int64_t k, uint32_t d) {
  uint64_t h = fmix64(fmix64(fmix64(seed0) ^ (uint64_t)k) ^ (uint64_t)d);
  int32_t q = (int32_t)(h >> 40) - (1 << 23);
  return __fmul_rn((float)q, 9.313225746154785e-10f);  // 2^-30, exact
}

__device__ __forceinline__ uint64_t hash_home(const Dev& s, int64_t key) {
  uint64_t h = ((uint64_t)key * 0x9E3779B97F4A7C15ull) >> (64 - s.hbits);
  return h & ~31ull;
}

__device__ __forceinline__ void raise_err(Ctl* ctl, int code) {
  atomicCAS(&ctl->err, 0, code);
  ctl->abort = 1;
}

// Warp-cooperative probe: all 32 lanes call with the same key; returns the
// entry index (>= 0) or -1 when absent.  A window of 32 aligned slots is read
// with one coalesced 256 B load; ballots find a match or an EMPTY slot.
__device__ __forceinline__ int32_t warp_find(const Dev& s, int64_t key, int lane) {
  uint64_t w = hash_home(s, key);
  for (int it = 0; it < (1 << 20); ++it) {
    uint64_t slot = (w + lane) & s.hmask;
    const uint64_t hw = s.hslot[slot];
    unsigned m = __ballot_sync(0xffffffffu, hs_is(hw, key));
    if (m) {
      const int32_t e = __shfl_sync(0xffffffffu, hs_val(hw), __ffs(m) - 1);
      HET_ASSERT(e >= 0 && e < s.Ecap);
      return e;
    }
    if (__ballot_sync(0xffffffffu, hw == HS_EMPTY)) return -1;
    w = (w + 32) & s.hmask;
  }
  return -1;
}

// As warp_find, also returning the slot (for an erase without a second probe).
__device__ __forceinline__ int32_t warp_find_slot(const Dev& s, int64_t key, int lane, uint64_t* slot_out) {
  uint64_t w = hash_home(s, key);
  for (int it = 0; it < (1 << 20); ++it) {
    uint64_t slot = (w + lane) & s.hmask;
    const uint64_t hw = s.hslot[slot];
    unsigned m = __ballot_sync(0xffffffffu, hs_is(hw, key));
    if (m) {
      int src = __ffs(m) - 1;
      *slot_out = __shfl_sync(0xffffffffu, slot, src);
      return __shfl_sync(0xffffffffu, hs_val(hw), src);
    }
    if (__ballot_sync(0xffffffffu, hw == HS_EMPTY)) return -1;
    w = (w + 32) & s.hmask;
  }
  return -1;
}

// As warp_find; on a miss also the slot warp_insert would claim (the first
// window holding a TOMB or EMPTY slot, its first TOMB else its first EMPTY)
// and that slot's word, so the insert is one CAS without a second probe.
__device__ __forceinline__ int32_t warp_find_cand(const Dev& s, int64_t key, int lane, uint64_t* cslot,
                                                  uint64_t* cword) {
  uint64_t w = hash_home(s, key);
  *cslot = ~0ull;
  for (int it = 0; it < (1 << 20); ++it) {
    uint64_t slot = (w + lane) & s.hmask;
    const uint64_t hw = s.hslot[slot];
    unsigned m = __ballot_sync(0xffffffffu, hs_is(hw, key));
    if (m) return __shfl_sync(0xffffffffu, hs_val(hw), __ffs(m) - 1);
    const unsigned me = __ballot_sync(0xffffffffu, hw == HS_EMPTY);
    if (*cslot == ~0ull) {
      const unsigned mt = __ballot_sync(0xffffffffu, hw == HS_TOMB);
      if (mt | me) {
        const int src = __ffs(mt ? mt : me) - 1;
        *cslot = __shfl_sync(0xffffffffu, slot, src);
        *cword = __shfl_sync(0xffffffffu, hw, src);
      }
    }
    if (me) return -1;
    w = (w + 32) & s.hmask;
  }
  return -1;
}

// Single-thread find (for many keys per warp): scans whole 32-slot windows
// (16 x 16 B loads) with the same stop rule as warp_find.
__device__ __forceinline__ int32_t thread_find_slot(const Dev& s, int64_t key, uint64_t* slot_out) {
  uint64_t w = hash_home(s, key);
  for (int it = 0; it < (1 << 20); ++it) {
    const ulonglong2* win = reinterpret_cast<const ulonglong2*>(s.hslot + w);
    bool empty = false;
    int hit = -1;
    int32_t val = -1;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const ulonglong2 v = win[q];
      if (hs_is(v.x, key)) { hit = 2 * q; val = hs_val(v.x); }
      if (hs_is(v.y, key)) { hit = 2 * q + 1; val = hs_val(v.y); }
      empty |= (v.x == HS_EMPTY) | (v.y == HS_EMPTY);
    }
    if (hit >= 0) {
      *slot_out = w + hit;
      return val;
    }
    if (empty) return -1;
    w = (w + 32) & s.hmask;
  }
  return -1;
}

// Warp-cooperative insert of a key known to be absent.  Claims the first
// EMPTY or TOMB slot in probe order with atomicCAS.
__device__ __forceinline__ void warp_insert(const Dev& s, int64_t key, int32_t entry, int lane) {
  uint64_t w = hash_home(s, key);
  for (;;) {
    uint64_t slot = (w + lane) & s.hmask;
    const uint64_t hw = s.hslot[slot];
    // prefer tombstones, so EMPTY slots (which end probes) are used up slowly
    unsigned mt = __ballot_sync(0xffffffffu, hw == HS_TOMB);
    unsigned me = __ballot_sync(0xffffffffu, hw == HS_EMPTY);
    for (int pass = 0; pass < 2; ++pass) {
      unsigned m = pass == 0 ? mt : me;
      while (m) {
        int src = __ffs(m) - 1;
        int ok = 0;
        if (lane == src) {   // key and entry in one CAS
          unsigned long long old = atomicCAS((unsigned long long*)&s.hslot[slot], (unsigned long long)hw,
                                             (unsigned long long)hs_pack(key, entry));
          if (old == (unsigned long long)hw) {
            if (hw == HS_TOMB) atomicSub(&s.ctl->n_tomb, 1);
            ok = 1;
          }
        }
        ok = __shfl_sync(0xffffffffu, ok, src);
        if (ok) return;
        m &= m - 1;
      }
    }
    w = (w + 32) & s.hmask;
  }
}

// Insert a key known to be absent at the candidate slot warp_find_cand
// returned (one CAS); a slot taken meanwhile falls back to warp_insert.
__device__ __forceinline__ void warp_insert_at(const Dev& s, int64_t key, int32_t entry, int lane, uint64_t cslot,
                                               uint64_t cword) {
  int ok = 0;
  if (lane == 0 && cslot != ~0ull) {
    const unsigned long long old = atomicCAS((unsigned long long*)&s.hslot[cslot], (unsigned long long)cword,
                                             (unsigned long long)hs_pack(key, entry));
    if (old == (unsigned long long)cword) {
      if (cword == HS_TOMB) atomicSub(&s.ctl->n_tomb, 1);
      ok = 1;
    }
  }
  if (!__shfl_sync(0xffffffffu, ok, 0)) warp_insert(s, key, entry, lane);
}

// Warp-cooperative delete: the key is present.
__device__ __forceinline__ void warp_erase(const Dev& s, int64_t key, int lane) {
  uint64_t w = hash_home(s, key);
  for (;;) {
    uint64_t slot = (w + lane) & s.hmask;
    const uint64_t hw = s.hslot[slot];
    unsigned m = __ballot_sync(0xffffffffu, hs_is(hw, key));
    if (m) {
      if (lane == __ffs(m) - 1) {
        s.hslot[slot] = HS_TOMB;
        atomicAdd(&s.ctl->n_tomb, 1);
      }
      return;
    }
    if (__ballot_sync(0xffffffffu, hw == HS_EMPTY)) return;  // not found (should not happen)
    w = (w + 32) & s.hmask;
  }
}

// move a key between LFU count bitmaps (oldc/newc = EP_FREE for none);
// dpop: block-local population deltas flushed by the caller
__device__ __forceinline__ void lfu_move(const Dev& s, int64_t key, uint32_t oldc, uint32_t newc, int* dpop) {
  if (s.lfu_cb == 0 || oldc == newc) return;
  int64_t w = key >> 5;
  uint32_t bit = 1u << (key & 31);
  int64_t blk = key >> LFU_BLK_SHIFT;
  if (oldc < (uint32_t)s.lfu_cb) {
    atomicAnd(&s.bm[(int64_t)oldc * s.bm_words + w], ~bit);
    atomicSub(&s.bcnt[(int64_t)oldc * s.nbk + blk], 1u);
    atomicSub(&s.bcnt2[(int64_t)oldc * s.nbk2 + (blk >> 6)], 1u);
    atomicSub(&dpop[oldc], 1);
  }
  if (newc < (uint32_t)s.lfu_cb) {
    atomicOr(&s.bm[(int64_t)newc * s.bm_words + w], bit);
    atomicAdd(&s.bcnt[(int64_t)newc * s.nbk + blk], 1u);
    atomicAdd(&s.bcnt2[(int64_t)newc * s.nbk2 + (blk >> 6)], 1u);
    atomicAdd(&dpop[newc], 1);
  }
}

__device__ __forceinline__ void dpop_init(int* dpop) {
  if (threadIdx.x < LFU_CB_MAX) dpop[threadIdx.x] = 0;
}
__device__ __forceinline__ void dpop_flush(const Dev& s, int* dpop) {
  if (s.lfu_cb && threadIdx.x < s.lfu_cb && dpop[threadIdx.x]) atomicAdd(&s.pop[threadIdx.x], dpop[threadIdx.x]);
}

// lookup -> update record of unique key u (warp-uniform call): the entry, its
// segment, c_c and dirty flag after the lookup (nothing changes them before
// the update) and the first four positions, so the update's segment reduce
// starts from two 16 B loads instead of a chain of dependent ones
__device__ __forceinline__ void write_urec(const Call& c, int u, int32_t e, int j0, int cnt, bool dirty,
                                           uint32_t cc, int pos_lane, int lane) {
  const int p0 = __shfl_sync(0xffffffffu, pos_lane, 0), p1 = __shfl_sync(0xffffffffu, pos_lane, 1);
  const int p2 = __shfl_sync(0xffffffffu, pos_lane, 2), p3 = __shfl_sync(0xffffffffu, pos_lane, 3);
  if (lane == 0 && e >= 0) {
    c.urec[u] = make_int4(e, j0, (int)((uint32_t)cnt | (dirty ? 0x80000000u : 0u)), (int)cc);
    c.upos[u] = make_int4(p0, p1, p2, p3);
  }
}

// rmode: the key run starting at sorted position r (warp-uniform): false if r
// is not the first position of its key.  Lane l loads composite r - 1 + l and
// the batch position of sorted r + l (both coalesced, in one round trip); a
// run longer than 31 is followed chunk by chunk.
__device__ __forceinline__ bool key_run(const Call& c, int r, int lane, int64_t* key, int* cnt, int* pos_lane) {
  const int n = c.n, pb = c.pbits;
  const int q = r - 1 + lane;
  const uint64_t w = (q >= 0 && q < n) ? __ldcg(&c.sortbuf0[q]) : ~0ull;
  const int pl = r + lane < n ? __ldcg(&c.perm[r + lane]) : 0;
  const uint64_t kl = w >> pb;
  const uint64_t k = __shfl_sync(0xffffffffu, kl, 1);
  const uint64_t kp = __shfl_sync(0xffffffffu, kl, 0);
  if (r > 0 && kp == k) return false;
  unsigned same = __ballot_sync(0xffffffffu, lane >= 1 && q < n && kl == k) >> 1;   // bit j: sorted r + j
  int len = __ffs(~same) - 1;                                                       // 1..31
  if (same == 0x7FFFFFFFu) {
    len = 31;
    for (int b = r + 31;; b += 32) {
      const int qq = b + lane;
      const bool eq = qq < n && (__ldcg(&c.sortbuf0[qq]) >> pb) == k;
      const unsigned m = __ballot_sync(0xffffffffu, eq);
      const int run = __ffs(~m) - 1;   // -1 when all 32 equal
      if (run < 0) { len += 32; continue; }
      len += run;
      break;
    }
  }
  *key = (int64_t)k;
  *cnt = len;
  *pos_lane = lane < len ? pl : 0;
  return true;
}

// LFU threshold (T, K*) for this step, one CTA (the last block of k_lookup_fused):
// T = the smallest count whose cumulative population reaches `need`, K* = the
// needT-th smallest key of count T.  Loads are issued in parallel: the 16
// populations by 16 lanes, the block counters of bitmap T in chunks of
// blockDim (coalesced, block-wide prefix), stopping at the chunk holding K*.
// ---------------------------------------------------------------- TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// one bulk (non-tensor) TMA copy global -> shared, completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// Wide rows (D >= 1024 and a multiple of 512): the fused paths move row bytes
// in their own kernels (k_mv_as, k_seg_as) instead of a warp per key.
__host__ __device__ __forceinline__ bool wide_rows(uint32_t D) {
  const uint32_t D4 = D >> 2;
  return D4 >= 256 && D4 % 128 == 0;
}

// warp-aggregated counter increment
__device__ __forceinline__ void warp_count(unsigned long long* c, bool pred) {
  unsigned m = __ballot_sync(__activemask(), pred);
  if (m && (threadIdx.x & 31) == (__ffs(__activemask()) - 1)) atomicAdd(c, (unsigned long long)__popc(m));
}

// ---------------------------------------------------------------- launchers
void launch_begin(const Dev& s, uint64_t t, int n, cudaStream_t st);
// dedup (K1): returns number of kernel launches issued
int launch_dedup(const Call& c, int n, int64_t R, int pbits, Ctl* ctl, cudaStream_t st);

// cache kernels (k_cache.cu)
void launch_init_shard(const Dev& s, cudaStream_t st);
void launch_reset_cache(const Dev& s, cudaStream_t st);
void launch_probe(const Dev& s, const Call& c, int n_max_units, cudaStream_t st);
void launch_sync_fetch_install_local(const Dev& s, const Call& c, int n_units, cudaStream_t st);
void launch_gather(const Dev& s, const Call& c, float* out, cudaStream_t st);
// K7/K8 for large batches: heavy keys streamed through a TMA ring on `side`
// (forked from and joined back into `st` with the two events), light keys on
// `st` concurrently.  Returns the number of kernel launches.
int launch_segreduce_apply(const Dev& s, const Call& c, const float* grads, float lr, int n, cudaStream_t st,
                           cudaStream_t side, cudaEvent_t fork, cudaEvent_t join);
int launch_evict_select(const Dev& s, void* evbuf, cudaStream_t st);
int launch_evict_apply_local(const Dev& s, void* evbuf, cudaStream_t st);
void launch_hash_rebuild(const Dev& s, cudaStream_t st);
// fused single-GPU step (k_fused.cu)
bool fused_ok(const Dev& s, int n);
int launch_pin_apply(const Dev& s, cudaStream_t st);
constexpr int FUSED_LOOKUP_MAX = 16384;   // N = 1: fused lookup/update up to this n
// evict: the previous fused update left listed victims (Ctl::ev_pending) --
// they are evicted by extra blocks of the same kernel; evbuf: EvBuf;
// p2pview: the exchange view at N > 1 (PUSH records), else nullptr
// compact: 1 writes unique/seg_off/U (rmode 0), 0 leaves the sorted
// composites for the rmode lookup (no serial tail).  lookup: 1 a lookup's
// dedup (the per-call begin), 0 an evict's, 2 het_prefetch's (no side effect
// on the cache state: only the sorted composites, perm and c.pref_bad)
int launch_dd_fused(const Dev& s, const Call& c, int n, int pbits, uint64_t t, int lookup, cudaStream_t st,
                    void* evbuf, const void* p2pview, bool evict, int compact);
// rmode: the compact lookup log (uniq, seg_off, dbg_status, dbg_inverse, dbg_U) for the debug export
void launch_compact_log(const Dev& s, const Call& c, cudaStream_t st);
int launch_evict_pending(const Dev& s, void* evbuf, const void* p2pview, cudaStream_t st);
// a lookup whose dedup het_prefetch already ran: the per-call begin (+ the deferred eviction)
int launch_begin_evict(const Dev& s, const Call& c, int n, uint64_t t, cudaStream_t st, void* evbuf,
                       const void* p2pview, bool evict);
// rmode dedup for 8192 < n <= 16384: one CTA, bucketed exact rank (+ the deferred eviction)
int launch_dd_bucket(const Dev& s, const Call& c, int n, int pbits, uint64_t t, int lookup, cudaStream_t st,
                     void* evbuf, const void* p2pview, bool evict);
constexpr int RMODE_MAX = 16384;   // rmode dedups serve n <= this
// prof: the handle when phase profiling is on (het_profile_enable), else nullptr
int launch_lookup_fused(const Dev& s, const Call& c, float* out, cudaStream_t st, void* prof = nullptr);
// N > 1, wide rows, rmode: the Get scatter out[perm[r]] = v[entry of r's key] of every sorted
// position r after the exchange round installed the rows (k_mv_as, scatter-only)
// resp: this worker's response records (REC floats each: 16 B header + the row), indexed by uslot;
// the rows refetched this round come from there, and their head position also writes v
int launch_scatter_wide(const Dev& s, const Call& c, float* out, cudaStream_t st, const float* resp, int64_t rec,
                        const int32_t* uslot);
// SMs left free by the cooperative kernels for NCCL's blocks at N > 1
// (= NCCL's maxCTAs and the peer-memory dense all-reduce grid; env HET_NCCL_CTAS, default 16)
int coop_sm_reserve();
int launch_update_fused(const Dev& s, const Call& c, const float* grads, float lr, void* evbuf, cudaStream_t st,
                        const void* p2pview = nullptr, void* prof = nullptr);

}  // namespace het
