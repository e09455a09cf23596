// Fused single-GPU step (N = 1, n <= 8192): three kernels per iteration.
//
//  k_dd_fused      rank-count stable sort of the (key, position) composites
//                  (K1); the last block to finish (atomic counter, no waiting)
//                  flags segment heads, block-scans them, writes
//                  unique/inverse/perm/seg_off and does the per-call begin
//                  (abort reset, clock, counters).
//  k_lookup_fused  warp per unique key: Cache.Find, CheckValid cond (1)+(2),
//                  LFU/LRU touch, fused Evict(k)+Fetch(k) / miss install, and
//                  Cache.Get scattered to every occurrence of the key (K2,
//                  K4/K5, K6).
//  k_update_fused  cooperative: warp per unique key does the ordered segment
//                  reduce + SGD + pending + clock (K7/K8)
//                  while block 0 derives this step's eviction threshold (with
//                  LFU count bitmaps the victims are exactly {count < T} plus
//                  the keys <= K* among count T; R9) and lists the
//                  bitmap blocks holding victims; after a grid sync the warps
//                  extract the victim keys (4096-key blocks), after another
//                  every victim is evicted by its own warp (Evict push W += p,
//                  c_g = max, delete, free; K9).  LRU / LFU
//                  fallback: generic selection then apply.  Hash rebuild,
//                  when requested.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "evict_dev.cuh"
#include "p2p_dev.cuh"
#include "het_mgpu.h"   // prof_begin / prof_end

namespace het {

// ---- optional timeline instrumentation (-DHET_TIMELINE): %globaltimer marks
// per kernel k: [0] min block start, [1] max block start, [2] max work end,
// [3] last-block tail start, [4] tail end
#ifdef HET_TIMELINE
// per-warp slots (no contention): g_tlw[mark][warp], read and reduced on the host
constexpr int TLW = 8192;
__device__ unsigned long long g_tlw[40 * TLW];   // rows 32..39: ad-hoc marks (TL_X)
__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TL_W(i) do { if ((threadIdx.x & 31) == 0) { int w_ = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; \
  if (w_ < TLW) g_tlw[(i) * TLW + w_] = tl_now(); } } while (0)
#define TL_MIN(i) TL_W(i)
#define TL_X(i) TL_W(32 + (i))
#define TL_MAX(i) TL_W(i)
extern "C" int het_debug_timeline(unsigned long long* out, int marks, int warps) {
  cudaDeviceSynchronize();
  if (out) cudaMemcpyFromSymbol(out, g_tlw, sizeof(unsigned long long) * (size_t)marks * TLW);
  cudaMemset((void*)0, 0, 0);
  static unsigned long long* zero = nullptr;
  if (!zero) zero = (unsigned long long*)calloc(40 * TLW, 8);
  cudaMemcpyToSymbol(g_tlw, zero, sizeof(unsigned long long) * 40 * TLW);
  (void)warps;
  return 0;
}
#else
#define TL_MIN(i) do {} while (0)
#define TL_X(i) do {} while (0)
#define TL_MAX(i) do {} while (0)
#endif

// Programmatic dependent launch (PDL): the next kernel of the step is
// launched while this one still runs (its blocks park in griddepcontrol.wait
// until this grid has completed and its writes are visible), hiding the
// launch gap between the three kernels.  HET_PDL=0 disables it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr int DDF_THREADS = 512;
constexpr int DDF_WARPS = DDF_THREADS / 32;
constexpr int DDF_ITEMS = 16;   // FUSED_MAX / DDF_THREADS (elements per lane in the finish)
constexpr int LK_WARPS = 8;
constexpr int UPD_THREADS = 256;
constexpr int UPD_WARPS = UPD_THREADS / 32;

__device__ __forceinline__ int block_scan_int(int x, int* warp_sums, int* tot) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_sums[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) warp_sums[lane] = w;
  }
  __syncthreads();
  int base = wid ? warp_sums[wid - 1] : 0;
  *tot = warp_sums[nw - 1];
  __syncthreads();
  return base + v - x;
}

// ------------------------------------------------------------------ K_dd
template <int RBE = 4>
__device__ __forceinline__ void evict_listed(const Dev& s, const EvBuf& b, const P2P* pp, int eb, int neb);

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// While the dedup ranks the keys, pull into L2 the lines the next kernels
// will wait on: per key of this block's 32 positions the hash window (two
// 128 B lines), the LFU count, c_g and the server row (a miss fetches it,
// P:439); block 0 also the LFU plan's counters and bitmap words around the
// previous step's threshold (the update's plan).  Hints only: no
// result depends on them.
__device__ __forceinline__ void prefetch_lookup_lines(const Dev& s, const uint32_t* kq, int n) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  if (p < n && wid < 8) {
    const int64_t key = (int64_t)kq[p];
    const bool own = key % s.world == s.rank;
    const int64_t row = key / s.world;
    if (wid < 2) prefetch_l2(s.hslot + hash_home(s, key) + 16 * wid);
    else if (wid == 2) { if (s.lfu_persist) prefetch_l2(s.count_by_key + key); }
    else if (wid == 3) { if (own) prefetch_l2(s.cg + row); }
    else if ((wid - 4) * 32 < (int)s.D && own) prefetch_l2(s.W + row * s.D + (wid - 4) * 32);
  }
  if (blockIdx.x == 0 && wid >= 8 && s.lfu_cb) {
    const Ctl* ctl = s.ctl;
    const uint32_t T = ctl->T;
    const int64_t ks = ctl->Kstar;
    if (T >= (uint32_t)s.lfu_cb || ks < 0 || ks >= s.R) return;
    const int64_t kblk = ks >> LFU_BLK_SHIFT;
    const int t = (wid - 8) * 32 + lane, nt = (DDF_WARPS - 8) * 32;
    if (t == 0) prefetch_l2(s.pop);
    for (int64_t i = (int64_t)t * 32; i < s.nbk2; i += (int64_t)nt * 32) prefetch_l2(s.bcnt2 + (int64_t)T * s.nbk2 + i);
    for (int64_t i = (int64_t)t * 32; i <= kblk + 64 && i < s.nbk; i += (int64_t)nt * 32)
      prefetch_l2(s.bcnt + (int64_t)T * s.nbk + i);
    const int64_t w0 = kblk << (LFU_BLK_SHIFT - 5);
    for (int64_t i = (int64_t)t * 32; i < 256; i += (int64_t)nt * 32)
      if (w0 + i < s.bm_words) prefetch_l2(s.bm + (int64_t)T * s.bm_words + w0 + i);
    // the words of every non-empty count-T block up to K*'s (the next
    // extraction reads them): one pass over the block counters
    const uint32_t* bc = s.bcnt + (int64_t)T * s.nbk;
    for (int64_t k = t; k <= kblk + 1 && k < s.nbk; k += nt)
      if (__ldcg(&bc[k]))
        for (int l = 0; l < 4; ++l)
          prefetch_l2(s.bm + (int64_t)T * s.bm_words + (k << (LFU_BLK_SHIFT - 5)) + 32 * l);
  }
}

// #{q in [q0, q1) : key_q <= m} (le) or < m, over whole 128-bit vectors
// (q0 a multiple of 4; keys past q1 in the last vector are padding above
// every key), two vectors and two partial sums per iteration
__device__ __forceinline__ int count_le(const uint4* __restrict__ k4, int q0, int q1, uint32_t m, bool le) {
  if (q0 >= q1) return 0;
  int c0 = 0, c1 = 0;
  const int v0 = q0 >> 2, v1 = (q1 + 3) >> 2;
  int v = v0;
  if (le) {
    for (; v + 1 < v1; v += 2) {
      const uint4 a = k4[v], b = k4[v + 1];
      c0 += (a.x <= m) + (a.y <= m) + (a.z <= m) + (a.w <= m);
      c1 += (b.x <= m) + (b.y <= m) + (b.z <= m) + (b.w <= m);
    }
    if (v < v1) { const uint4 a = k4[v]; c0 += (a.x <= m) + (a.y <= m) + (a.z <= m) + (a.w <= m); }
  } else {
    for (; v + 1 < v1; v += 2) {
      const uint4 a = k4[v], b = k4[v + 1];
      c0 += (a.x < m) + (a.y < m) + (a.z < m) + (a.w < m);
      c1 += (b.x < m) + (b.y < m) + (b.z < m) + (b.w < m);
    }
    if (v < v1) { const uint4 a = k4[v]; c0 += (a.x < m) + (a.y < m) + (a.z < m) + (a.w < m); }
  }
  return c0 + c1;
}

// per-call begin (block 0, thread 0): clock, sequence, counters, abort reset
__device__ __forceinline__ void dd_begin(const Dev& s, const Call& c, int n, uint64_t t, int lookup, int bad,
                                         int compact) {
  Ctl* ctl = s.ctl;
  if (lookup) {
    if (t == CLOCK_AUTO) { t = ctl->t_auto; ctl->t_auto = t + 1; }
    ctl->t_cur = t;
    ctl->lk_seq = ctl->lk_seq + 1;
    s.cnt[C_LOOKUPS] += 1;
    s.cnt[C_KEYS] += (unsigned long long)n;
  }
  ctl->abort = 0;
  ctl->nsel = 0;              // the update's victim list (its extraction blocks append)
  if (!compact) ctl->U = n;   // rmode: every sorted position is a work item of the lookup
  if (bad) { raise_err(ctl, 2 /*HET_ERR_KEY_RANGE*/); ctl->U = 0; c.seg_off[0] = 0; }
}

// rmode dedup (K1): the stable sort position of every occurrence, r(p) =
// #{q : key_q < key_p} + #{q < p : key_q == key_p}, counted over the 32-bit
// keys in shared memory (R15: keys < 2^32), four per 128-bit load; block b
// ranks positions [32b, 32b + 32), its warps split the q range.  Writes the
// sorted composites (key << pbits | p) and perm; the lookup reads key runs.
__device__ __forceinline__ void dd_rank_rmode(const int64_t* __restrict__ keys, int n, int pbits, const Dev& s,
                                              const Call& c, uint64_t t, int lookup, uint32_t* kq,
                                              int (*part)[32]) {
  int bad = 0;
  {  // all key loads of this thread in flight at once
    int64_t kk[DDF_ITEMS];
#pragma unroll
    for (int i = 0; i < DDF_ITEMS; ++i) {
      const int q = threadIdx.x + i * DDF_THREADS;
      kk[i] = q < n ? __ldg(&keys[q]) : 0;
    }
#pragma unroll
    for (int i = 0; i < DDF_ITEMS; ++i) {
      const int q = threadIdx.x + i * DDF_THREADS;
      if (q < n) {
        if (kk[i] < 0 || kk[i] >= s.R) bad = 1;
        kq[q] = (uint32_t)kk[i];
      }
    }
    const int npad = (n + 3) & ~3;   // pad to whole 128-bit loads with a key above every real one
    if (threadIdx.x < npad - n) kq[n + threadIdx.x] = 0xFFFFFFFFu;
  }
  bad = __syncthreads_or(bad);
  TL_MAX(1);
  if (!bad && lookup) prefetch_lookup_lines(s, kq, n);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (lookup == 2) *c.pref_bad = bad;   // het_prefetch: the consuming lookup raises it
    else dd_begin(s, c, n, t, lookup, bad, 0);
  }
  if (bad) return;
  TL_MAX(3);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  const uint32_t mine = p < n ? kq[p] : 0xFFFFFFFFu;
  const int per = (((n + DDF_WARPS - 1) / DDF_WARPS) + 3) & ~3;
  const int q0 = min(n, wid * per), q1 = min(n, q0 + per);
  const int pmin = blockIdx.x * 32, pmax = pmin + 31;
  const uint4* k4 = reinterpret_cast<const uint4*>(kq);
  int cnt = 0;
  if (q1 <= pmin) {           // every q before every p of the block: key_q <= key_p (q1 = q0 + per: whole vectors)
    cnt = count_le(k4, q0, q1, mine, true);
  } else if (q0 > pmax) {     // every q after every p: key_q < key_p (ranges end on a multiple of 4 or
    cnt = count_le(k4, q0, q1, mine, false);   // in the padding, which never counts)
  } else {                    // the range meets the block's own positions: before / among / after them
    const int a = max(q0, min(q1, pmin)), z = max(a, min(q1, pmax + 1));
    cnt = count_le(k4, q0, a, mine, true);       // q0 and pmin are multiples of 4
    for (int q = a; q < z; ++q) {
      const uint32_t x = kq[q];
      cnt += (x < mine) || (x == mine && q < p);
    }
    cnt += count_le(k4, z, q1, mine, false);     // pmax + 1 is a multiple of 4; padding never counts
  }
  part[wid][lane] = cnt;
  __syncthreads();
  TL_MAX(5);
  if (wid == 0 && p < n) {
    int r = 0;
#pragma unroll
    for (int w = 0; w < DDF_WARPS; ++w) r += part[w][lane];
    HET_ASSERT(r >= 0 && r < n);
    c.sortbuf0[r] = ((uint64_t)mine << pbits) | (uint64_t)p;
    c.perm[r] = p;                 // stable position grouping
  }
  TL_MAX(2);
}

// blocks [0, ndd): the dedup; blocks [ndd, gridDim.x): the overflow eviction
// the previous update listed (deferred, see k_update_fused) -- independent
// work, side by side
__global__ void __launch_bounds__(DDF_THREADS)
k_dd_fused(const int64_t* __restrict__ keys, int n, int pbits, Dev s, Call c, uint64_t t, int lookup, EvBuf eb,
           P2P pm, int push, int ndd, int compact) {
  pdl_trigger();
  if ((int)blockIdx.x >= ndd) {
    evict_listed<8>(s, eb, push ? &pm : nullptr, blockIdx.x - ndd, gridDim.x - ndd);
    return;
  }
  extern __shared__ __align__(16) uint64_t comp[];
  __shared__ int part[DDF_WARPS][32];
  __shared__ int warp_sums[32];
  __shared__ int s_last;
  Ctl* ctl = s.ctl;
  TL_MIN(0);
  if (!compact) {
    dd_rank_rmode(keys, n, pbits, s, c, t, lookup, reinterpret_cast<uint32_t*>(comp), part);
    return;
  }
  int bad = 0;
  {  // all key loads of this thread in flight at once
    int64_t kk[DDF_ITEMS];
#pragma unroll
    for (int i = 0; i < DDF_ITEMS; ++i) {
      const int q = threadIdx.x + i * DDF_THREADS;
      kk[i] = q < n ? __ldg(&keys[q]) : 0;
    }
#pragma unroll
    for (int i = 0; i < DDF_ITEMS; ++i) {
      const int q = threadIdx.x + i * DDF_THREADS;
      if (q < n) {
        if (kk[i] < 0 || kk[i] >= s.R) bad = 1;
        comp[q] = ((uint64_t)kk[i] << pbits) | (uint64_t)q;
      }
    }
  }
  bad = __syncthreads_or(bad);
  if (blockIdx.x == 0 && threadIdx.x == 0) dd_begin(s, c, n, t, lookup, bad, 1);   // overlapped with the rank work
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  if (!bad) {
    const uint64_t mine = p < n ? comp[p] : ~0ull;
    const int per = (n + DDF_WARPS - 1) / DDF_WARPS;
    const int q0 = wid * per, q1 = min(n, q0 + per);
    int cnt = 0;
#pragma unroll 8
    for (int q = q0; q < q1; ++q) cnt += comp[q] < mine;
    part[wid][lane] = cnt;
    __syncthreads();
    if (wid == 0 && p < n) {
      int r = 0;
#pragma unroll
      for (int w = 0; w < DDF_WARPS; ++w) r += part[w][lane];
      c.sortbuf0[r] = mine;
      c.perm[r] = p;                 // stable position grouping, written here (distributed)
    }
  }
  TL_MAX(2);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->dd_done, 1) == ndd - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  TL_MAX(3);
  // ---- last block: head flags / scan / outputs
  if (threadIdx.x == 0) ctl->dd_done = 0;
  if (bad) return;
  // warp w owns the contiguous segment [w*seg, (w+1)*seg) of the sorted
  // composites: coalesced loads, head flags by ballot, one cross-warp prefix
  const uint64_t* sorted = c.sortbuf0;
  const int seg = ((n + DDF_WARPS - 1) / DDF_WARPS + 31) & ~31;
  const int s0 = wid * seg, s1 = min(n, s0 + seg);
  uint64_t x[DDF_ITEMS];
  unsigned hm[DDF_ITEMS];
  uint64_t prevlast = (s0 > 0 && s0 <= n) ? __ldcg(&sorted[s0 - 1]) : ~0ull;
#pragma unroll
  for (int i = 0; i < DDF_ITEMS; ++i) {
    const int j = s0 + i * 32 + lane;
    x[i] = j < s1 ? __ldcg(&sorted[j]) : ~0ull;
  }
  int wcnt = 0;
  TL_MAX(5);
#pragma unroll
  for (int i = 0; i < DDF_ITEMS; ++i) {
    const int j = s0 + i * 32 + lane;
    uint64_t prev = __shfl_up_sync(0xffffffffu, x[i], 1);
    if (lane == 0) prev = prevlast;
    const bool head = j < s1 && (j == 0 || (x[i] >> pbits) != (prev >> pbits));
    hm[i] = __ballot_sync(0xffffffffu, head);
    wcnt += __popc(hm[i]);
    prevlast = __shfl_sync(0xffffffffu, x[i], 31);
  }
  if (lane == 0) warp_sums[wid] = wcnt;
  __syncthreads();
  int base = 0, tot = 0;
  for (int w = 0; w < DDF_WARPS; ++w) {
    const int v = warp_sums[w];
    if (w < wid) base += v;
    tot += v;
  }
  TL_MAX(6);
  int run = base - 1;                 // unique index of the last head seen
#pragma unroll
  for (int i = 0; i < DDF_ITEMS; ++i) {
    const int j = s0 + i * 32 + lane;
    const int u = run + __popc(hm[i] & ((2u << lane) - 1u));   // heads up to and including lane
    if (j < s1 && ((hm[i] >> lane) & 1u)) {   // perm: rank blocks; inverse: the lookup kernel
      c.uniq[u] = (int64_t)(x[i] >> pbits);
      c.seg_off[u] = j;
    }
    run += __popc(hm[i]);
  }
  if (threadIdx.x == 0) { c.seg_off[tot] = n; ctl->U = tot; }
  TL_MAX(4);
}

// ------------------------------------------------------------------ K_look
struct Plan {          // an eviction plan (shared memory of the block that derives it)
  int emode;           // 0 none, 1 LFU count bitmaps, 2 generic selection
  int rebuild;         // hash rebuild requested (tombstones > S/8)
  uint32_t T;          // threshold count
  uint32_t lowmask;    // counts < T with residents (all of them victims)
  int64_t Kstar;       // largest victim key of count T
  int64_t needT;       // victims among count T
  int64_t need;        // |cache| - C
  int64_t ftop;        // free-stack top (victim i frees into fstack[ftop + i])
};

__device__ void lfu_threshold(const Dev& s, int* warp_sums_i, long long* warp_sums, int64_t need, Plan* pl) {
  __shared__ int s_T;
  __shared__ long long s_needT;
  __shared__ long long s_blk, s_before;
  __shared__ int s_done;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    long long pc = lane < s.lfu_cb ? (long long)__ldcg(&s.pop[lane]) : 0;
    long long incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long excl = incl - pc;
    const unsigned hit = __ballot_sync(0xffffffffu, lane < s.lfu_cb && excl < need && incl >= need);
    const unsigned nonempty = __ballot_sync(0xffffffffu, pc > 0);
    if (lane == 0) {
      pl->emode = 2;                        // until K* is found below
      s_T = hit ? __ffs(hit) - 1 : -1;
    }
    if (hit && lane == __ffs(hit) - 1) {
      s_needT = need - excl;
      pl->lowmask = nonempty & ((1u << lane) - 1u);
    }
  }
  __syncthreads();
  TL_MAX(7);
  if (s_T < 0) return;
  const int T = s_T;
  const int64_t needT = s_needT;
  const uint32_t* bc = s.bcnt + (int64_t)T * s.nbk;
  const uint32_t* bm = s.bm + (int64_t)T * s.bm_words;
  if (threadIdx.x == 0) { s_done = 0; s_blk = -1; }
  __syncthreads();
  // level 2: the 64-block super-block holding the needT-th bit (chunks of blockDim)
  __shared__ long long s_sb, s_sbbefore;
  const uint32_t* bc2 = s.bcnt2 + (int64_t)T * s.nbk2;
  long long carry = 0;
  for (int64_t base = 0; base < s.nbk2 && !s_done; base += blockDim.x) {
    const int64_t k = base + threadIdx.x;
    const long long x = k < s.nbk2 ? (long long)__ldcg(&bc2[k]) : 0;
    long long tot;
    const long long ex = carry + block_excl_scan64(x, warp_sums, &tot);
    if (x > 0 && ex < needT && ex + x >= needT) { s_sb = k; s_sbbefore = ex; s_done = 1; }
    carry += tot;
    __syncthreads();
  }
  TL_MAX(24);
  // level 1: the block inside the super-block (64 counters, one warp)
  if (s_done && threadIdx.x < 32) {
    const int64_t b0 = s_sb << 6;
    const int64_t k0 = b0 + 2 * threadIdx.x;
    const long long x0 = k0 < s.nbk ? (long long)__ldcg(&bc[k0]) : 0;
    const long long x1 = k0 + 1 < s.nbk ? (long long)__ldcg(&bc[k0 + 1]) : 0;
    long long incl = x0 + x1;
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)threadIdx.x >= o) incl += y;
    }
    const long long ex = s_sbbefore + incl - x0 - x1;
    if (x0 > 0 && ex < needT && ex + x0 >= needT) { s_blk = k0; s_before = ex; }
    if (x1 > 0 && ex + x0 < needT && ex + x0 + x1 >= needT) { s_blk = k0 + 1; s_before = ex + x0; }
  }
  __syncthreads();
  TL_MAX(25);
  if (s_blk < 0) return;
  if (threadIdx.x < 32) {
    const int64_t blk = s_blk;
    const int64_t want = needT - s_before;      // 1-based rank inside the block
    uint32_t w[4];
    int cl = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int64_t wi = (blk << (LFU_BLK_SHIFT - 5)) + lane * 4 + q;
      w[q] = wi < s.bm_words ? __ldcg(&bm[wi]) : 0u;
      cl += __popc(w[q]);
    }
    int incl = cl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int excl = incl - cl;
    if (excl < want && incl >= want) {
      int r = (int)(want - excl);               // r-th set bit among this lane's 4 words
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int pc = __popc(w[q]);
        if (r <= pc) {
          uint32_t bits = w[q];
          for (int kk = 1; kk < r; ++kk) bits &= bits - 1;
          int64_t key = (((blk << (LFU_BLK_SHIFT - 5)) + lane * 4 + q) << 5) + (__ffs(bits) - 1);
          pl->Kstar = key;
          pl->T = (uint32_t)T;
          pl->needT = needT;
          pl->emode = 1;
          break;
        }
        r -= pc;
      }
    }
  }
}

__global__ void __launch_bounds__(LK_WARPS * 32)
k_lookup_fused(Dev s, Call c, float* __restrict__ out, int agg) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned bc[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ int s_nmiss, s_base;
  __shared__ uint32_t s_minp;
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  if (threadIdx.x == 0) { s_nmiss = 0; s_minp = 0xFFFFFFFFu; }
  dpop_init(dpop);
  TL_MIN(8);
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * LK_WARPS + (threadIdx.x >> 5);   // rmode: sorted position r
  const int U = c.rmode ? c.n : ctl->U;
  const int D4 = s.D >> 2;
  bool live = !ctl->abort && u < U;
  // ---- phase A (warp per unique key): Find, CheckValid, touch; with agg (large
  // n: thousands of misses) a miss takes a slot of the block's free-entry
  // reservation -- one atomic per block between the phases instead of one per miss
  int64_t key = 0;
  int j0 = 0, cnt = 0, pos_lane = 0, moff = 0;
  int32_t e = -1;
  uint8_t st = ST_HIT;
  uint32_t ecs = 0, ecc = 0, cntk = 0, gpre = 0, mprim = 0;
  if (live && c.rmode) {
    // one window: lane l holds sorted composite r - 1 + l and the position of
    // sorted r + l -- the head test, the key, its run length and positions
    live = key_run(c, u, lane, &key, &cnt, &pos_lane);
    j0 = u;
    if (!live && lane == 0) c.urec[u].x = -1;   // not a key's first sorted position: no work for the update
  } else if (live) {
    key = c.uniq[u];
    j0 = c.seg_off[u];
    cnt = c.seg_off[u + 1] - j0;
    pos_lane = lane < cnt ? c.perm[j0 + lane] : 0;
  }
  // rows of at most 128 floats live in registers, one float4 per lane: the
  // server row (a miss or refetch installs it) is loaded with the probe and
  // the cached row (a hit returns it) as soon as the probe ends, so neither
  // waits for the decisions
  const bool reg = D4 <= 32;
  const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 wrow = zero4, vrow = zero4;
  uint64_t cslot = ~0ull, cword = 0;   // a miss's insert slot, from the probe
  if (live) {
    if (lane == 0 && s.lfu_persist) cntk = s.count_by_key[key];
    if (lane == 1) gpre = s.cg[key];
    if (reg && lane < D4) wrow = __ldcg(reinterpret_cast<const float4*>(s.W + key * s.D) + lane);
    e = warp_find_cand(s, key, lane, &cslot, &cword);
    if (reg && e >= 0 && lane < D4) vrow = __ldcg(reinterpret_cast<const float4*>(s.v + (int64_t)e * s.D) + lane);
    gpre = __shfl_sync(0xffffffffu, gpre, 1);
    TL_MAX(13);
    st = ST_MISS;
    if (e >= 0) { ecs = s.cs[e]; ecc = s.cc[e]; }
    if (lane == 0) {
      // light-LFU: a pinned entry skips the frequency maintenance
      const uint32_t oldc = (e >= 0 && s.policy == 0) ? s.eprim[e] : 0u;
      const bool pinned = oldc == EP_PIN;
      if (s.lfu_persist && !pinned) { cntk += 1; s.count_by_key[key] = cntk; }
      if (e >= 0) {
        if (s.s == S_INF) st = ST_HIT;                       // R4
        else if (ecc - ecs > s.s) st = ST_EXP1;              // cond (1)
        else st = (gpre <= ecc || gpre - ecc <= s.s) ? ST_HIT : ST_EXP2;   // cond (2)
        if (s.policy == 0) {                                 // L6
          if (!pinned) {
            uint32_t newc = s.lfu_persist ? cntk : oldc + 1;
            s.eprim[e] = newc;
            lfu_move(s, key, oldc, newc, dpop);
            pin_candidate(s, key, e, newc);
          }
        } else {
          s.eprim[e] = (uint32_t)ctl->t_cur;
        }
      } else {
        mprim = s.policy == 0 ? (s.lfu_persist ? cntk : 1u) : (uint32_t)ctl->t_cur;
        if (agg) {
          moff = atomicAdd(&s_nmiss, 1);
          atomicMin(&s_minp, mprim);
        } else {
          moff = atomicSub(&ctl->ftop, 1) - 1;      // the entry's free-stack index
          atomicMin(&ctl->min_install, mprim);
          TL_MAX(28);
        }
      }
      c.status[u] = st;
      atomicAdd(&bc[st == ST_HIT ? 0 : st == ST_EXP1 ? 1 : st == ST_EXP2 ? 2 : 3], 1u);
    }
    st = __shfl_sync(0xffffffffu, st, 0);
    moff = __shfl_sync(0xffffffffu, moff, 0);
  }
  if (agg) {                                 // uniform per launch
    __syncthreads();
    if (threadIdx.x == 0 && s_nmiss) {       // the block's misses: one free-stack pop, one min_install
      s_base = atomicSub(&ctl->ftop, s_nmiss);
      atomicMin(&ctl->min_install, s_minp);
    }
    __syncthreads();
  }
  // ---- phase B: sync push / fetch / install, Get scatter
  if (live) {
    float4* Wr = reinterpret_cast<float4*>(s.W + key * s.D);
    uint32_t ucc = ecc;              // the entry's c_c and dirty flag as the update will find them
    bool udirty = ecc > ecs;
    if (st != ST_HIT) {
      uint32_t g = gpre;   // c_g[key]: only this warp touches the key's server row and clock
      if (st != ST_MISS) {
        if (ecc > ecs) {  // dirty sync push (L4): W += p, c_g = max
          const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
          if (reg) {
            if (lane < D4) { wrow = f4add_(wrow, pr[lane]); Wr[lane] = wrow; }
          } else {
            for (int d = lane; d < D4; d += 32) Wr[d] = f4add_(Wr[d], pr[d]);
          }
          g = g > ecc ? g : ecc;
          if (lane == 0) s.cg[key] = g;
        }
      } else {          // miss: the reserved free entry + hash insert
        const int idx = agg ? s_base - 1 - moff : moff;
        if (idx < 0) {
          if (lane == 0) raise_err(ctl, 4 /*HET_ERR_CAPACITY*/);
          e = -1;
        } else {
          HET_ASSERT(idx >= 0 && idx < s.Ecap);
          e = s.fstack[idx];
          HET_ASSERT(e >= 0 && e < s.Ecap);
          TL_MAX(29);
          warp_insert_at(s, key, e, lane, cslot, cword);
          TL_MAX(30);
          if (lane == 0) {
            s.ekey[e] = key;
            s.eprim[e] = mprim;
            if (s.policy == 0) { lfu_move(s, key, EP_FREE, mprim, dpop); pin_candidate(s, key, e, mprim); }
          }
        }
      }
      if (e >= 0) {     // L5: v = W, c_s = c_c = c_g
        float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
        if (reg) {
          if (lane < D4) vr[lane] = wrow;
        } else {
          for (int d = lane; d < D4; d += 32) vr[d] = Wr[d];
        }
        if (lane == 0) { s.cs[e] = g; s.cc[e] = g; }
        ucc = g;
        udirty = false;
      }
      vrow = wrow;
    }
    TL_MAX(14);
    for (int k = lane; k < cnt; k += 32) c.inverse[k < 32 ? pos_lane : c.perm[j0 + k]] = u;
    write_urec(c, u, e, j0, cnt, udirty, ucc, pos_lane, lane);
    if (e >= 0 && reg) {
      if (lane == 0) c.uentry[u] = e;
      // L7 Get, scattered to the occurrences of the key (128-bit stores)
      float4* o4 = reinterpret_cast<float4*>(out);
      for (int kb = 0; kb < cnt; kb += 32) {
        const int src = kb == 0 ? pos_lane : (kb + lane < cnt ? c.perm[j0 + kb + lane] : 0);
        const int m = min(32, cnt - kb);
        for (int k = 0; k < m; ++k) {
          const int pos = __shfl_sync(0xffffffffu, src, k);
          if (lane < D4) __stcs(o4 + (int64_t)pos * D4 + lane, vrow);
        }
      }
    } else if (e >= 0) {
      if (lane == 0) c.uentry[u] = e;
      // L7 Get, scattered to the occurrences of the key (128-bit stores)
      const float4* vr = reinterpret_cast<const float4*>(s.v + (int64_t)e * s.D);
      float4* o4 = reinterpret_cast<float4*>(out);
      for (int d = lane; d - lane < D4; d += 32) {
        float4 val = d < D4 ? vr[d] : make_float4(0.f, 0.f, 0.f, 0.f);
        if (d == lane) { __syncwarp(); TL_MAX(15); }
        for (int kb = 0; kb < cnt; kb += 32) {
          const int src = kb == 0 ? pos_lane : (kb + lane < cnt ? c.perm[j0 + kb + lane] : 0);
          const int m = min(32, cnt - kb);
          for (int k = 0; k < m; ++k) {
            int pos = __shfl_sync(0xffffffffu, src, k);
            if (d < D4) __stcs(o4 + (int64_t)pos * D4 + d, val);
          }
        }
      }
    }
  }
  TL_MAX(10);
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP1], (unsigned long long)bc[1]);
    if (bc[2]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[2]);
    if (bc[3]) atomicAdd(&s.cnt[C_MISSES], (unsigned long long)bc[3]);
    if (c.rmode) {
      const unsigned nu = bc[0] + bc[1] + bc[2] + bc[3];   // heads of this block
      if (nu) atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)nu);
    } else if (blockIdx.x == 0 && !ctl->abort) {
      atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)U);
    }
  }
  // light-LFU (R27): the last block applies this lookup's promotions
  if (s.pin_thr) {
    __shared__ int s_lastpin;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_lastpin = atomicAdd(&ctl->lk_done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (s_lastpin) {
      __threadfence();
      pin_apply_block(s);
      if (threadIdx.x == 0) ctl->lk_done = 0;
    }
  }
}

// ------------------------------------------------------------------ K_look, wide rows
// D >= 1024 (BASELINE configs[4], D = 4096: 16 KB rows).  G = 0 (the fused
// rmode path): a warp per sorted position takes every decision of
// k_lookup_fused (Find, CheckValid, touch, sync push clock, install
// allocation) and leaves the row moves to k_mv_as (flags in ucnt).  G > 0
// (unsorted-unique mode): G = D/512 warps per key, the first takes the
// decisions, then after a block barrier each warp moves its 512-column
// slice: the Evict push W += p, the Fetch v = W and the Get scatter.
struct LkMeta { int64_t key; int32_t e; int32_t j0; int32_t cnt; uint32_t g; uint8_t st; uint8_t push; };

__global__ void __launch_bounds__(LK_WARPS * 32)
k_lookup_wide(Dev s, Call c, float* __restrict__ out, int G) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned bc[4];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ LkMeta meta[LK_WARPS];
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  dpop_init(dpop);
  __syncthreads();
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int GG = G > 0 ? G : 1;   // G == 0: one warp per key, decisions only
  const int grp = wib / GG, gw = wib % GG;
  const int u = blockIdx.x * (LK_WARPS / GG) + grp;   // rmode: sorted position r
  const int U = c.rmode ? c.n : ctl->U;
  const bool live = !ctl->abort && u < U;
  bool head = true;
  int64_t key = 0;
  int j0 = 0, cnt = 0, pl = 0;
  if (live && gw == 0) {
    if (c.rmode) {
      head = key_run(c, u, lane, &key, &cnt, &pl);
      j0 = u;
      if (!head && lane == 0) { c.urec[u].x = -1; meta[grp].e = -1; }
    } else {
      key = c.uniq[u];
      j0 = c.seg_off[u];
      cnt = c.seg_off[u + 1] - j0;
      pl = lane < cnt ? c.perm[j0 + lane] : 0;
    }
  }
  if (live && gw == 0 && head) {
    uint32_t cntk = 0, gpre = 0;
    if (lane == 0 && s.lfu_persist) cntk = s.count_by_key[key];
    if (lane == 1 && s.s != S_INF) gpre = s.cg[key];
    int32_t e = warp_find(s, key, lane);
    gpre = __shfl_sync(0xffffffffu, gpre, 1);
    uint8_t st = ST_MISS;
    uint32_t ecs = 0, ecc = 0;
    if (e >= 0) { ecs = s.cs[e]; ecc = s.cc[e]; }
    if (lane == 0) {
      const uint32_t oldc = (e >= 0 && s.policy == 0) ? s.eprim[e] : 0u;
      const bool pinned = oldc == EP_PIN;
      if (s.lfu_persist && !pinned) { cntk += 1; s.count_by_key[key] = cntk; }
      if (e >= 0) {
        if (s.s == S_INF) st = ST_HIT;                       // R4
        else if (ecc - ecs > s.s) st = ST_EXP1;              // cond (1)
        else st = (gpre <= ecc || gpre - ecc <= s.s) ? ST_HIT : ST_EXP2;   // cond (2)
        if (s.policy == 0) {                                 // L6
          if (!pinned) {
            uint32_t newc = s.lfu_persist ? cntk : oldc + 1;
            s.eprim[e] = newc;
            lfu_move(s, key, oldc, newc, dpop);
            pin_candidate(s, key, e, newc);
          }
        } else {
          s.eprim[e] = (uint32_t)ctl->t_cur;
        }
      }
      c.status[u] = st;
      atomicAdd(&bc[st == ST_HIT ? 0 : st == ST_EXP1 ? 1 : st == ST_EXP2 ? 2 : 3], 1u);
    }
    st = __shfl_sync(0xffffffffu, st, 0);
    uint32_t g = gpre;
    bool push = false;
    if (st != ST_HIT) {
      if (s.s == S_INF || st == ST_MISS) g = s.cg[key];
      if (st != ST_MISS) {
        if (ecc > ecs) {            // dirty sync push (L4): c_g = max (rows below)
          push = true;
          g = g > ecc ? g : ecc;
          if (lane == 0) s.cg[key] = g;
        }
      } else {                      // miss: free entry + hash insert
        int32_t idx = 0;
        if (lane == 0) idx = atomicSub(&ctl->ftop, 1) - 1;
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx < 0) {
          if (lane == 0) raise_err(ctl, 4 /*HET_ERR_CAPACITY*/);
          e = -1;
        } else {
          HET_ASSERT(idx >= 0 && idx < s.Ecap);
          e = s.fstack[idx];
          HET_ASSERT(e >= 0 && e < s.Ecap);
          warp_insert(s, key, e, lane);
          if (lane == 0) {
            s.ekey[e] = key;
            uint32_t prim = s.policy == 0 ? (s.lfu_persist ? cntk : 1u) : (uint32_t)ctl->t_cur;
            s.eprim[e] = prim;
            if (s.policy == 0) { lfu_move(s, key, EP_FREE, prim, dpop); pin_candidate(s, key, e, prim); }
            atomicMin(&ctl->min_install, prim);
          }
        }
      }
      if (e >= 0 && lane == 0) { s.cs[e] = g; s.cc[e] = g; }   // L5 clocks (rows below)
    }
    for (int k = lane; k < cnt; k += 32) c.inverse[c.perm[j0 + k]] = u;
    write_urec(c, u, e, j0, cnt, st == ST_HIT && ecc > ecs, st == ST_HIT ? ecc : g, pl, lane);
    if (lane == 0) {
      if (e >= 0) c.uentry[u] = e;
      meta[grp] = LkMeta{key, e, j0, cnt, g, st, (uint8_t)push};
      if (G == 0) {   // decisions only: the row moves are k_lookup_wide_mv's (key, fetch | push << 1)
        c.uniq[u] = key;
        c.ucnt[u] = (e >= 0 ? (st != ST_HIT ? 1 : 0) | (push ? 2 : 0) : 0) | (e >= 0 ? 4 : 0);
      }
    }
  }
  if (G == 0 && live && c.rmode && gw == 0 && !head && lane == 0) c.ucnt[u] = 0;
  __syncthreads();
  if (live && G > 0) {
    const LkMeta mt = meta[grp];
    const int D4 = s.D >> 2;
    const int d0 = gw * (D4 / G), d1 = d0 + D4 / G;
    if (mt.e >= 0) {
      float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)mt.e * s.D);
      if (mt.st != ST_HIT) {
        float4* Wr = reinterpret_cast<float4*>(s.W + mt.key * s.D);
        const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)mt.e * s.D);
        for (int d = d0 + lane; d < d1; d += 32) {
          float4 w = Wr[d];
          if (mt.push) { w = f4add_(w, pr[d]); Wr[d] = w; }   // Evict push
          vr[d] = w;                                           // Fetch
        }
      }
      // L7 Get: this warp's slice of the row to every occurrence (128-bit stores)
      float4* o4 = reinterpret_cast<float4*>(out);
      for (int kb = 0; kb < mt.cnt; kb += 32) {
        const int src = kb + lane < mt.cnt ? c.perm[mt.j0 + kb + lane] : 0;
        const int m = min(32, mt.cnt - kb);
        for (int d = d0 + lane; d < d1; d += 32) {
          const float4 val = vr[d];
          for (int k = 0; k < m; ++k) __stcs(o4 + (int64_t)__shfl_sync(0xffffffffu, src, k) * D4 + d, val);
        }
      }
    }
  }
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (bc[0]) atomicAdd(&s.cnt[C_HITS], (unsigned long long)bc[0]);
    if (bc[1]) atomicAdd(&s.cnt[C_EXP1], (unsigned long long)bc[1]);
    if (bc[2]) atomicAdd(&s.cnt[C_EXP2], (unsigned long long)bc[2]);
    if (bc[3]) atomicAdd(&s.cnt[C_MISSES], (unsigned long long)bc[3]);
    if (c.rmode) {
      const unsigned nu = bc[0] + bc[1] + bc[2] + bc[3];   // heads of this block
      if (nu) atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)nu);
    } else if (blockIdx.x == 0 && !ctl->abort) {
      atomicAdd(&s.cnt[C_UNIQUE], (unsigned long long)U);
    }
  }
  // light-LFU (R27): the last block applies this lookup's promotions
  if (s.pin_thr) {
    __shared__ int s_lastpin;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_lastpin = atomicAdd(&ctl->lk_done, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (s_lastpin) {
      __threadfence();
      pin_apply_block(s);
      if (threadIdx.x == 0) ctl->lk_done = 0;
    }
  }
}

// ------------------------------------------------------------------ K_upd
// Evict push of one resident entry at N = 1 (warp-cooperative) + delete + free
// push != nullptr (N > 1): the Evict push goes to the owner's inbox, carried
// by the next exchange round; otherwise the local server applies it now
// vi: the victim's export index; fpos: the free-stack slot its entry goes to
// (the caller reserved [ftop, ftop + victims) once: no per-victim atomics on
// the shared cursors; tombstones are counted per block in *s_tomb)
template <int RBE = 4>   // float4 columns per lane in flight in the push (wide rows)
__device__ __forceinline__ void evict_entry(const Dev& s, const EvBuf& b, int32_t e, int64_t key, uint64_t slot,
                                            int lane, int* dpop, unsigned* s_dirty, unsigned* s_ev,
                                            unsigned* s_tomb, int vi, int64_t fpos, const P2P* push = nullptr) {
  const uint32_t ecs = s.cs[e], ecc = s.cc[e], prim = s.eprim[e];
  const bool dirty = ecc > ecs;
  const int D4 = s.D >> 2;
  if (dirty && push) {
    push_record(s, *push, e, key, ecc, lane);
  } else if (dirty) {
    float4* Wr = reinterpret_cast<float4*>(s.W + key * s.D);
    const float4* pr = reinterpret_cast<const float4*>(s.p + (int64_t)e * s.D);
    for (int d0 = lane; d0 < D4; d0 += 32 * RBE) {   // RBE columns per lane in flight (wide rows)
      float4 w[RBE], x[RBE];
#pragma unroll
      for (int b = 0; b < RBE; ++b) if (d0 + 32 * b < D4) { w[b] = Wr[d0 + 32 * b]; x[b] = pr[d0 + 32 * b]; }
#pragma unroll
      for (int b = 0; b < RBE; ++b) if (d0 + 32 * b < D4) Wr[d0 + 32 * b] = f4add_(w[b], x[b]);
    }
  }
  if (lane == 0) {
    if (push && dirty) atomicAdd(&s.cnt[C_BEMB_TX], 16ull + 4ull * s.D);
    if (dirty && !push) { uint32_t g = s.cg[key]; s.cg[key] = g > ecc ? g : ecc; }
    s.hslot[slot] = HS_TOMB;
    atomicAdd(s_tomb, 1u);
    b.vkeys[vi] = key;
    b.vdirty[vi] = dirty ? 1 : 0;
    if (s.policy == 0) lfu_move(s, key, prim, EP_FREE, dpop);
    unpin_count(s, prim);
    s.eprim[e] = EP_FREE;
    s.ekey[e] = -1;
    HET_ASSERT(fpos >= 0 && fpos < s.Ecap && e >= 0 && e < s.Ecap);
    s.fstack[fpos] = e;
    atomicAdd(s_ev, 1u);
    if (dirty) atomicAdd(s_dirty, 1u);
  }
}

__device__ __forceinline__ void segreduce_key(const Dev& s, const Call& c, const float4* __restrict__ G4, float lr,
                                              int u, int lane, float4* mystg, uint64_t* bar, uint32_t& phase,
                                              int stage_rows) {
  // the lookup's record: entry, segment, c_c, dirty flag and the first four
  // positions -- two independent 16 B loads start the key's work
  const int4 rec = __ldcg(&c.urec[u]);
  const int4 p4 = __ldcg(&c.upos[u]);
  const int32_t e = rec.x;
  if (e < 0) return;   // rmode: not a key's first sorted position
  const int j0 = rec.y;
  const int cnt = rec.z & 0x7FFFFFFF;
  const bool dirty = rec.z < 0;
  const uint32_t ecc = (uint32_t)rec.w;
  const int D4 = s.D >> 2;
  const float nlr = -lr;
  float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
  float4* pr = reinterpret_cast<float4*>(s.p + (int64_t)e * s.D);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (stage_rows > 0 && cnt > 4) {
    const int pos_lane = lane < cnt ? __ldg(&c.perm[j0 + lane]) : 0;
    float4* accrow = mystg + (size_t)stage_rows * D4;
    const uint32_t rowbytes = s.D * 4;
    for (int kb = 0; kb < cnt; kb += stage_rows) {
      const int m = min(stage_rows, cnt - kb);
      const int src = kb == 0 ? pos_lane : (kb + lane < cnt ? __ldg(&c.perm[j0 + kb + lane]) : 0);
      __syncwarp();
      fence_proxy_async();
      if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)m * rowbytes);
      __syncwarp();
      if (lane < m) bulk_g2s(mystg + (size_t)lane * D4, G4 + (int64_t)src * D4, rowbytes, bar);
      mbar_wait(bar, phase);
      phase ^= 1;
      for (int d = lane; d < D4; d += 32) {
        float4 a = kb ? accrow[d] : zero;
        for (int k = 0; k < m; ++k) a = f4add_(a, mystg[(size_t)k * D4 + d]);
        accrow[d] = a;
      }
    }
    __syncwarp();
    for (int d = lane; d < D4; d += 32) {
      float4 acc = accrow[d];
      float4 dl = make_float4(__fmul_rn(nlr, acc.x), __fmul_rn(nlr, acc.y), __fmul_rn(nlr, acc.z),
                              __fmul_rn(nlr, acc.w));
      vr[d] = f4add_(vr[d], dl);
      pr[d] = f4add_(dirty ? pr[d] : zero, dl);
    }
  } else if (cnt <= 4) {
    // the common case: every occurrence row, v and p in flight at once
    for (int d = lane; d - lane < D4; d += 32) {
      const bool act = d < D4;
      float4 vv = act ? vr[d] : zero;
      float4 pp = (act && dirty) ? pr[d] : zero;
      float4 g0 = zero, g1 = zero, g2 = zero, g3 = zero;
      if (act) {
        g0 = __ldcs(G4 + (int64_t)p4.x * D4 + d);
        if (cnt > 1) g1 = __ldcs(G4 + (int64_t)p4.y * D4 + d);
        if (cnt > 2) g2 = __ldcs(G4 + (int64_t)p4.z * D4 + d);
        if (cnt > 3) g3 = __ldcs(G4 + (int64_t)p4.w * D4 + d);
      }
      float4 acc = f4add_(zero, g0);                 // +0.0f, then ascending position (R11)
      if (cnt > 1) acc = f4add_(acc, g1);
      if (cnt > 2) acc = f4add_(acc, g2);
      if (cnt > 3) acc = f4add_(acc, g3);
      if (act) {
        float4 dl = make_float4(__fmul_rn(nlr, acc.x), __fmul_rn(nlr, acc.y), __fmul_rn(nlr, acc.z),
                                __fmul_rn(nlr, acc.w));
        vr[d] = f4add_(vv, dl);
        pr[d] = f4add_(pp, dl);
      }
    }
  } else {
    const int pos_lane = lane < cnt ? __ldg(&c.perm[j0 + lane]) : 0;
    for (int d = lane; d - lane < D4; d += 32) {
      const bool act = d < D4;
      float4 vv = act ? vr[d] : zero;
      float4 pp = (act && dirty) ? pr[d] : zero;
      float4 acc = zero;
      for (int kb = 0; kb < cnt; kb += 32) {
        const int src = kb == 0 ? pos_lane : (kb + lane < cnt ? __ldg(&c.perm[j0 + kb + lane]) : 0);
        const int m = min(32, cnt - kb);
        int k = 0;
        for (; k + 4 <= m; k += 4) {
          int p0 = __shfl_sync(0xffffffffu, src, k), p1 = __shfl_sync(0xffffffffu, src, k + 1);
          int p2 = __shfl_sync(0xffffffffu, src, k + 2), p3 = __shfl_sync(0xffffffffu, src, k + 3);
          if (act) {
            float4 g0 = __ldcs(G4 + (int64_t)p0 * D4 + d), g1 = __ldcs(G4 + (int64_t)p1 * D4 + d);
            float4 g2 = __ldcs(G4 + (int64_t)p2 * D4 + d), g3 = __ldcs(G4 + (int64_t)p3 * D4 + d);
            acc = f4add_(acc, g0); acc = f4add_(acc, g1); acc = f4add_(acc, g2); acc = f4add_(acc, g3);
          }
        }
        for (; k < m; ++k) {
          int p0 = __shfl_sync(0xffffffffu, src, k);
          if (act) acc = f4add_(acc, __ldcs(G4 + (int64_t)p0 * D4 + d));
        }
      }
      if (act) {
        float4 dl = make_float4(__fmul_rn(nlr, acc.x), __fmul_rn(nlr, acc.y), __fmul_rn(nlr, acc.z),
                                __fmul_rn(nlr, acc.w));
        vr[d] = f4add_(vv, dl);
        pr[d] = f4add_(pp, dl);
      }
    }
  }
  if (lane == 0) s.cc[e] = ecc + 1;
}

// Wide rows (D >= 1024, BASELINE configs[4]: 16 KB rows): the ordered
// segment reduce + SGD + pending of every (key, slice) item in its own kernel
// (k_seg_as) ahead of the cooperative update, which then steps the clocks.
// Every thread is its own copy pipeline.
// Measured on B200 (tools/tma_probe.cu, random row chunks of an 8 GB table):
// one warp issuing cp.async.bulk copies completes ~2.7 M copies/s whatever
// the ring depth (1 KB copies: 2.8 GB/s per warp), so a key with 128
// occurrences is ~48 us of copy issue on one warp, and bulk copies need
// many issuing warps; plain loads reach the same plateau (~4 TB/s for 2 KB
// chunks) but a warp holds only what its registers hold.  Here a CTA of 128
// threads owns a (128 x F float4)-column slice of its items, thread t the
// float4 columns t + 128 j: each thread issues 16-byte cp.async copies
// (LDGSTS: no register cost, no depth cap) of its columns of every
// occurrence row, v and p into its own
// ring of row slots in shared memory, several stages ahead, one commit group
// per stage, and consumes the oldest stage after cp.async.wait_group -- its
// own copies, so no barrier.  A stage is <= CH occurrence rows of one
// item (+ v, p with its last); the sum runs in ascending position with the
// accumulator carried across the item's stages (+0.0f first, R11), then
// v += -lr*acc, p = (dirty ? p : +0) + -lr*acc (R13).  Items (key, slice) are
// dealt as (key group, slice) = (b / S, b % S) over the CTAs.  The kernel is
// issue-bound (ncu: 'wait' and 'selected' lead the stalls), so the ring, the
// columns per thread and the CTAs per SM were chosen by measurement; a
// dynamic (atomic) deal of the units and per-warp pipelines measured slower.
constexpr int AS_T = 128;     // threads per CTA (x F float4 columns: the slice)
constexpr int AS_QMAX = 7;    // stages in flight per thread (cp.async.wait_group immediates 0..6)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16s(uint32_t dst, const void* src) {   // dst: shared address
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait(int n) {   // at most n of this thread's groups still pending
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
  }
}

// The stage sequence of this CTA (identical in every thread; lane-dependent
// only in the lane's own record of the current batch of 32 keys).
// MV: the lookup's row moves (k_mv_as): heads with an entry, one stage per item.
template <bool MV, int CH>
struct AsWalk {
  int U, Q, u0;
  int4 rec, p4;
  int64_t key;
  int fl;
  unsigned live;
  bool valid, dirty;
  int l, e, j0, cnt, c0, m, flag;
  int64_t ikey;
  int hd, ihd;   // MV: bit 0 the key's head, bits 1..: the output row (lane's / item's)
  bool scat = false;   // MV: scatter only (N > 1: the rows are installed)
  const int32_t* uslot = nullptr;   // scat: each key's response slot (owner * CAPS + slot)

  __device__ __forceinline__ void load(const Call& c, int lane) {
    for (;;) {
      if (u0 >= U) { valid = false; return; }
      const int u = u0 + lane * Q;
      rec = make_int4(-1, 0, 0, 0);
      p4 = make_int4(0, 0, 0, 0);
      key = 0;
      fl = 0;
      hd = 0;
      if (u < U) {
        if (MV) {   // sorted position u: its output row perm[u] and its key's head inverse[perm[u]]
          const int p = __ldcg(&c.perm[u]);
          const int h = __ldcg(&c.inverse[p]);
          if (scat) {   // scatter only: every position of a key with an entry copies its row to out
            rec = __ldcg(&c.urec[h]);
            fl = rec.x >= 0 ? 4 : 0;
            const uint8_t st = __ldcg(&c.status[h]);
            if (fl && (st == ST_MISS || st == ST_EXP1 || st == ST_EXP2)) {   // refetched this round:
              fl |= 8;                                                        // the row is in its response
              key = __ldcg(&uslot[h]);
            }
            hd = (h == u ? 1 : 0) | (p << 1);
          } else {
          fl = __ldcg(&c.ucnt[h]);
          if ((fl & 4) && (!(fl & 2) || h == u)) {   // a push moves all its rows from the head
            rec = __ldcg(&c.urec[h]);
            key = __ldcg(&c.uniq[h]);
            if (fl & 2) p4 = __ldcg(&c.upos[h]);
            hd = (h == u ? 1 : 0) | (p << 1);
          } else {
            fl = 0;
          }
          }
        } else {
          rec = __ldcg(&c.urec[u]);
          p4 = __ldcg(&c.upos[u]);
        }
      }
      // rmode non-heads / capacity failures / past the end carry no work
      live = __ballot_sync(0xffffffffu, MV ? (fl & 4) != 0 : rec.x >= 0);
      if (live) { valid = true; return; }
      u0 += 32 * Q;
    }
  }
  __device__ __forceinline__ void item() {
    l = __ffs(live) - 1;
    live &= live - 1;
    e = __shfl_sync(0xffffffffu, rec.x, l);
    j0 = __shfl_sync(0xffffffffu, rec.y, l);
    const int z = __shfl_sync(0xffffffffu, rec.z, l);
    cnt = z & 0x7FFFFFFF;
    dirty = z < 0;
    c0 = 0;
    m = MV ? cnt : min(CH, cnt);
    if (MV) {
      flag = __shfl_sync(0xffffffffu, fl, l);
      ikey = __shfl_sync(0xffffffffu, key, l);
      ihd = __shfl_sync(0xffffffffu, hd, l);
    }
    valid = true;
  }
  __device__ __forceinline__ void init(const Call& c, int U_, int Q_, int q, int lane) {
    U = U_; Q = Q_; u0 = q;
    load(c, lane);
    if (valid) item();
  }
  __device__ __forceinline__ void next(const Call& c, int lane) {
    if (!MV && c0 + m < cnt) { c0 += m; m = min(CH, cnt - c0); return; }
    if (!live) {
      u0 += 32 * Q;
      load(c, lane);
      if (!valid) return;
    }
    item();
  }
  __device__ __forceinline__ bool last() const { return MV || c0 + m == cnt; }
  __device__ __forceinline__ int rows() const {
    return MV ? 1 + ((flag & 2) ? 1 : 0) : m + (c0 + m == cnt ? 1 + (dirty ? 1 : 0) : 0);
  }
  // this lane's occurrence position of the stage's row `lane` (rows < 32)
  __device__ __forceinline__ int pos_lane(const Call& c, int lane, int kb) const {
    if (cnt <= 4) {
      const int px = __shfl_sync(0xffffffffu, p4.x, l), py = __shfl_sync(0xffffffffu, p4.y, l);
      const int pz = __shfl_sync(0xffffffffu, p4.z, l), pw = __shfl_sync(0xffffffffu, p4.w, l);
      return lane == 0 ? px : lane == 1 ? py : lane == 2 ? pz : pw;
    }
    return c0 + kb + lane < cnt ? __ldg(&c.perm[j0 + c0 + kb + lane]) : 0;
  }
};

template <int RING>
__device__ __forceinline__ int ring_at(int x) {
  static_assert((RING & (RING - 1)) == 0, "ring size: a power of two");
  return x & (RING - 1);
}

template <int RING, int F, int CH>
__global__ void __launch_bounds__(AS_T) k_seg_as(Dev s, Call c, const float* __restrict__ G, float lr) {
  extern __shared__ __align__(16) float4 ring[];   // [RING][F][AS_T]: row slot r, column j of thread t at (r * F + j) * AS_T + t
  const uint32_t sbase = smem_u32(ring) + threadIdx.x * 16;
  pdl_wait();
  TL_X(5);
  const Ctl* ctl = s.ctl;
  const int U = ctl->abort ? 0 : (c.rmode ? c.n : ctl->U);
  const int D4 = s.D >> 2, S = D4 / (AS_T * F);
  const int Q = (int)gridDim.x / S;
  if ((int)blockIdx.x >= Q * S) return;
  const int t = threadIdx.x, lane = t & 31;
  const int col4 = ((int)blockIdx.x % S) * (AS_T * F) + t;
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const float4* v4 = reinterpret_cast<const float4*>(s.v);
  const float4* p4g = reinterpret_cast<const float4*>(s.p);
  AsWalk<false, CH> iw, cw;   // issue and consume positions in the same stage sequence
  iw.init(c, U, Q, (int)blockIdx.x / S, lane);
  cw.init(c, U, Q, (int)blockIdx.x / S, lane);
  int inflight = 0, used = 0, head = 0, tail = 0;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float nlr = -lr;
  float4 acc[F];
#pragma unroll
  for (int j = 0; j < F; ++j) acc[j] = zero;
  while (cw.valid) {
    while (iw.valid && inflight < AS_QMAX) {
      const int rows = iw.rows();
      if (used + rows > RING) break;
      const int pos = iw.pos_lane(c, lane, 0);
      for (int q = 0; q < iw.m; ++q) {
        const int64_t pq = __shfl_sync(0xffffffffu, pos, q);
        const float4* g = G4 + pq * D4 + col4;
        const uint32_t d = sbase + ring_at<RING>(head + q) * (F * AS_T * 16);
#pragma unroll
        for (int j = 0; j < F; ++j) cp_async16s(d + j * (AS_T * 16), g + j * AS_T);
      }
      if (iw.last()) {
        const uint32_t dv = sbase + ring_at<RING>(head + iw.m) * (F * AS_T * 16);
        const uint32_t dp = sbase + ring_at<RING>(head + iw.m + 1) * (F * AS_T * 16);
#pragma unroll
        for (int j = 0; j < F; ++j) {
          cp_async16s(dv + j * (AS_T * 16), v4 + (int64_t)iw.e * D4 + col4 + j * AS_T);
          if (iw.dirty) cp_async16s(dp + j * (AS_T * 16), p4g + (int64_t)iw.e * D4 + col4 + j * AS_T);
        }
      }
      cp_async_commit();
      ++inflight;
      used += rows;
      head = ring_at<RING>(head + rows);
      iw.next(c, lane);
    }
    cp_async_wait(inflight - 1);   // the oldest stage has landed
    for (int q = 0; q < cw.m; ++q) {   // ascending position
      const float4* r = ring + ring_at<RING>(tail + q) * (F * AS_T) + t;
#pragma unroll
      for (int j = 0; j < F; ++j) acc[j] = f4add_(acc[j], r[j * AS_T]);
    }
    if (cw.last()) {
      const float4* rv = ring + ring_at<RING>(tail + cw.m) * (F * AS_T) + t;
      const float4* rp = ring + ring_at<RING>(tail + cw.m + 1) * (F * AS_T) + t;
      float4* vo = reinterpret_cast<float4*>(s.v) + (int64_t)cw.e * D4 + col4;
      float4* po = reinterpret_cast<float4*>(s.p) + (int64_t)cw.e * D4 + col4;
#pragma unroll
      for (int j = 0; j < F; ++j) {
        const float4 vv = rv[j * AS_T];
        const float4 pp = cw.dirty ? rp[j * AS_T] : zero;
        const float4 dl = make_float4(__fmul_rn(nlr, acc[j].x), __fmul_rn(nlr, acc[j].y), __fmul_rn(nlr, acc[j].z),
                                      __fmul_rn(nlr, acc[j].w));
        vo[j * AS_T] = f4add_(vv, dl);
        po[j * AS_T] = f4add_(pp, dl);
        acc[j] = zero;
      }
    }
    const int rows = cw.rows();
    --inflight;
    used -= rows;
    tail = ring_at<RING>(tail + rows);
    cw.next(c, lane);
  }
  TL_X(6);
}

// The wide lookup's row moves (after k_lookup_wide with G = 0), the same
// per-thread pipelines over (sorted position, slice) items, so a key with
// 128 occurrences is spread over as many CTAs as any other positions (dealt
// per key, its scatter was the kernel's tail: ncu timeline, p90 26 us, max
// 52 us).  A position stages its key's source slice -- v[e] for a hit,
// W[key] for a refetch or miss -- and writes its own output row (Get,
// P:474); the key's head position also writes v[e] = W[key] (Fetch).
// No other position writes what another reads: W is read-only here except
// under the Evict push W += p, whose key is moved whole by its
// head (p[e] staged too, W[key] = v[e] = W + p, then every occurrence).
template <int RING, int F>
__global__ void __launch_bounds__(AS_T) k_mv_as(Dev s, Call c, float* __restrict__ out, int scat,
                                                const float* __restrict__ resp, int64_t rec,
                                                const int32_t* __restrict__ uslot) {
  extern __shared__ __align__(16) float4 ring[];
  const uint32_t sbase = smem_u32(ring) + threadIdx.x * 16;
  pdl_wait();
  const int U = s.ctl->abort ? 0 : c.n;   // rmode
  const int D4 = s.D >> 2, S = D4 / (AS_T * F);
  const int Q = (int)gridDim.x / S;
  if ((int)blockIdx.x >= Q * S) return;
  const int t = threadIdx.x, lane = t & 31;
  const int col4 = ((int)blockIdx.x % S) * (AS_T * F) + t;
  float4* W4 = reinterpret_cast<float4*>(s.W);
  float4* v4 = reinterpret_cast<float4*>(s.v);
  const float4* p4g = reinterpret_cast<const float4*>(s.p);
  float4* o4 = reinterpret_cast<float4*>(out);
  AsWalk<true, 1> iw, cw;
  iw.scat = cw.scat = scat != 0;
  iw.uslot = cw.uslot = uslot;
  iw.init(c, U, Q, (int)blockIdx.x / S, lane);
  cw.init(c, U, Q, (int)blockIdx.x / S, lane);
  int inflight = 0, used = 0, head = 0, tail = 0;
  while (cw.valid) {
    while (iw.valid && inflight < AS_QMAX) {
      const int rows = iw.rows();
      if (used + rows > RING) break;
      const float4* src = (iw.flag & 8)   ? reinterpret_cast<const float4*>(resp + iw.ikey * rec + 4)
                          : (iw.flag & 1) ? W4 + iw.ikey * D4
                                          : v4 + (int64_t)iw.e * D4;
      const uint32_t d0 = sbase + head * (F * AS_T * 16), d1 = sbase + ring_at<RING>(head + 1) * (F * AS_T * 16);
#pragma unroll
      for (int j = 0; j < F; ++j) {
        cp_async16s(d0 + j * (AS_T * 16), src + col4 + j * AS_T);
        if (iw.flag & 2) cp_async16s(d1 + j * (AS_T * 16), p4g + (int64_t)iw.e * D4 + col4 + j * AS_T);
      }
      cp_async_commit();
      ++inflight;
      used += rows;
      head = ring_at<RING>(head + rows);
      iw.next(c, lane);
    }
    cp_async_wait(inflight - 1);
    float4 w[F];
    const float4* r0 = ring + tail * (F * AS_T) + t;
    const float4* r1 = ring + ring_at<RING>(tail + 1) * (F * AS_T) + t;
    const bool head = cw.ihd & 1;
#pragma unroll
    for (int j = 0; j < F; ++j) {
      w[j] = r0[j * AS_T];
      if (cw.flag & 2) w[j] = f4add_(w[j], r1[j * AS_T]);
      if (head && (cw.flag & 9)) v4[(int64_t)cw.e * D4 + col4 + j * AS_T] = w[j];   // Fetch: v = the row
      if (cw.flag & 2) W4[cw.ikey * D4 + col4 + j * AS_T] = w[j];
    }
    if (cw.flag & 2) {   // push (the head's item): every occurrence
      for (int kb = 0; kb < cw.cnt; kb += 32) {
        const int pos = cw.pos_lane(c, lane, kb);
        const int mm = min(32, cw.cnt - kb);
        for (int q = 0; q < mm; ++q) {
          float4* o = o4 + (int64_t)__shfl_sync(0xffffffffu, pos, q) * D4 + col4;
#pragma unroll
          for (int j = 0; j < F; ++j) __stcs(o + j * AS_T, w[j]);
        }
      }
    } else {             // this position's row
      float4* o = o4 + (int64_t)(cw.ihd >> 1) * D4 + col4;
#pragma unroll
      for (int j = 0; j < F; ++j) __stcs(o + j * AS_T, w[j]);
    }
    const int rows = cw.rows();
    --inflight;
    used -= rows;
    tail = ring_at<RING>(tail + rows);
    cw.next(c, lane);
  }
  TL_X(7);
}

// ring rows, float4 columns per thread, rows per stage, CTAs per SM (macros: sweeps)
// (measured best of 11 pairs at BASELINE configs[4], tools/gpu_jobs.sh wide_sweep)
#ifndef AS_SEG_R
#define AS_SEG_R 16
#define AS_SEG_F 2
#define AS_SEG_C 8
#define AS_SEG_N 3
#endif
#ifndef AS_MV_R
#define AS_MV_R 4
#define AS_MV_F 2
#define AS_MV_N 12
#endif
constexpr int AS_SEG[4] = {AS_SEG_R, AS_SEG_F, AS_SEG_C, AS_SEG_N};   // 16 x 2 x 2 KB = 64 KB per CTA
constexpr int AS_MV[3] = {AS_MV_R, AS_MV_F, AS_MV_N};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// LFU bitmap path: the victim keys -- every resident key of count c < T (the
// counts in lowmask) and the keys <= K* of count T -- appended to vsel.
// Warp (gw, nw) takes chunks of 16 bitmap blocks (4096 keys each): one block
// counter per lane, then the words of up to XB non-empty blocks at once
// (4 words per lane each) and one vsel reservation for them.
constexpr int XCH = 16;   // bitmap blocks per extraction chunk
constexpr int XB = 4;     // non-empty blocks whose words are in flight at once (the batch logic assumes 4)
__device__ __forceinline__ void extract_victims(const Dev& s, const EvBuf& b, const Plan& pl, int gw, int nw,
                                                int lane) {
  Ctl* ctl = s.ctl;
  const uint32_t T = pl.T;
  const int64_t Kstar = pl.Kstar;
  const uint32_t lowmask = pl.lowmask;
  const int64_t kblk = Kstar >> LFU_BLK_SHIFT;
  const int64_t nch_full = (s.nbk + XCH - 1) / XCH, nch_T = (kblk + XCH) / XCH;
  int64_t total = nch_T;                       // chunks: counts < T in lowmask (all blocks), then count T
  for (uint32_t cc = 0; cc < T; ++cc) if ((lowmask >> cc) & 1) total += nch_full;
  for (int64_t it = gw; it < total; it += nw) {
    uint32_t cc = T;
    int64_t ch = it;
    for (uint32_t x = 0; x < T; ++x) {
      if (!((lowmask >> x) & 1)) continue;
      if (ch < nch_full) { cc = x; break; }
      ch -= nch_full;
    }
    const int64_t nb = cc < T ? s.nbk : kblk + 1;
    const int64_t blk_l = ch * XCH + lane;
    const uint32_t bcv = (lane < XCH && blk_l < nb) ? __ldcg(&s.bcnt[(int64_t)cc * s.nbk + blk_l]) : 0u;
    unsigned nz = __ballot_sync(0xffffffffu, bcv != 0);
    TL_MAX(9);
    const uint32_t* bm = s.bm + (int64_t)cc * s.bm_words;
    while (nz) {
      int32_t blk[XB];   // fixed slots (registers): block of batch slot j, or -1
#pragma unroll
      for (int j = 0; j < XB; ++j) {
        blk[j] = nz ? (int32_t)(ch * XCH) + (__ffs(nz) - 1) : -1;
        nz &= nz - 1;
      }
      const int nbat = (blk[XB - 1] >= 0) ? XB : (blk[2] >= 0 ? 3 : (blk[1] >= 0 ? 2 : 1));
      uint32_t w[XB][4];
#pragma unroll
      for (int j = 0; j < XB; ++j)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t wi = j < nbat ? ((int64_t)blk[j] << (LFU_BLK_SHIFT - 5)) + lane * 4 + r : 0;
          w[j][r] = (j < nbat && wi < s.bm_words) ? __ldcg(&bm[wi]) : 0u;
        }
      TL_MAX(4);
      int cl[XB], incl[XB], tot = 0;
#pragma unroll
      for (int j = 0; j < XB; ++j) {
        cl[j] = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (cc == T && j < nbat) {   // keep keys <= K*
            const int64_t k0 = (((int64_t)blk[j] << (LFU_BLK_SHIFT - 5)) + lane * 4 + r) << 5;
            if (k0 > Kstar) w[j][r] = 0;
            else if (k0 + 31 > Kstar) w[j][r] &= (1u << (Kstar - k0 + 1)) - 1u;
          }
          cl[j] += __popc(w[j][r]);
        }
        incl[j] = cl[j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl[j], o);
          if (lane >= o) incl[j] += y;
        }
        tot += __shfl_sync(0xffffffffu, incl[j], 31);
      }
      TL_MAX(17);
      if (!tot) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(&ctl->nsel, tot);
      base = __shfl_sync(0xffffffffu, base, 0);
      TL_MAX(31);
      // the batch's victims fill vsel[base, base + tot), lane by lane in key order
#pragma unroll
      for (int j = 0; j < XB; ++j) {
        int pos = base + incl[j] - cl[j];
        base += __shfl_sync(0xffffffffu, incl[j], 31);
        if (j >= nbat) continue;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          uint32_t bits = w[j][r];
          const int64_t kb = (((int64_t)blk[j] << (LFU_BLK_SHIFT - 5)) + lane * 4 + r) << 5;
          while (bits) {
            b.vsel[pos++] = kb + (__ffs(bits) - 1);
            bits &= bits - 1;
          }
        }
      }
      TL_MAX(6);
    }
  }
}

// This step's eviction plan from the cache state after the lookup (counts
// final: L6 precedes U3).  Deterministic: block 0 and every
// extraction block derive the same plan from the same state, so the
// extraction needs no hand-off from block 0.
__device__ __forceinline__ void make_plan(const Dev& s, bool abort, Plan* pl) {
  __shared__ long long warp_sums[32];
  __shared__ int warp_sums_i[32];
  Ctl* ctl = s.ctl;
  if (threadIdx.x == 0) {
    const int64_t ftop = __ldcg(&ctl->ftop);
    const int64_t res = s.Ecap - ftop;
    const int64_t need = res - s.C;
    const bool none = abort || need <= 0;
    pl->need = none ? 0 : need;
    pl->ftop = ftop;
    pl->emode = none ? 0 : ((s.policy == 0 && s.lfu_cb && need < res) ? 1 : 2);
    pl->rebuild = (int64_t)__ldcg(&ctl->n_tomb) > ((int64_t)s.hmask + 1) / 8;
    pl->T = 0; pl->lowmask = 0; pl->Kstar = -1; pl->needT = 0;
  }
  __syncthreads();
  if (pl->emode == 1) lfu_threshold(s, warp_sums_i, warp_sums, pl->need, pl);
  __syncthreads();
}

// The deferred overflow eviction: victim i of the listed vsel[0, ev_nsel) by
// warp (gw, nw) of the blocks given this work -- find, Evict push (W += p,
// c_g = max; N > 1: PUSH record to the owner's inbox), delete, free into
// fstack[ev_ftop0 + i].  Called by the first kernel of the call
// after the update (no other kernel touches the cache in between).
template <int RBE>
__device__ __forceinline__ void evict_listed(const Dev& s, const EvBuf& b, const P2P* pp, int eb, int neb) {
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty, s_ev, s_tomb;
  __shared__ int s_go, s_last;
  Ctl* ctl = s.ctl;
  dpop_init(dpop);
  if (threadIdx.x == 0) { s_dirty = 0; s_ev = 0; s_tomb = 0; s_go = __ldcg(&ctl->ev_pending); }
  __syncthreads();
  if (!s_go) return;   // uniform per block
  const int lane = threadIdx.x & 31;
  const int nwb = blockDim.x >> 5;
  const int gw = eb * nwb + (threadIdx.x >> 5), nw = neb * nwb;
  const int nsel = __ldcg(&ctl->ev_nsel);
  const int64_t ftop0 = __ldcg(&ctl->ev_ftop0);
  for (int i = gw; i < nsel; i += nw) {
    const int64_t key = __ldcg(&b.vsel[i]);
    uint64_t slot = 0;
    const int32_t e = warp_find_slot(s, key, lane, &slot);
    if (e >= 0) evict_entry<RBE>(s, b, e, key, slot, lane, dpop, &s_dirty, &s_ev, &s_tomb, i, ftop0 + i, pp);
    else if (lane == 0) raise_err(ctl, 3 /*HET_ERR_PROTOCOL: a listed victim is not resident*/);
  }
  TL_MAX(12);
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (s_ev) atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)s_ev);
    if (s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
    if (s_tomb) atomicAdd(&ctl->n_tomb, (int)s_tomb);
    if (eb == 0) ctl->ftop = (int32_t)(ftop0 + nsel);   // nothing else moves the free stack in this kernel
    __threadfence();
    s_last = atomicAdd(&ctl->ev_done, 1) == neb - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) { ctl->ev_done = 0; ctl->ev_pending = 0; }
}

// the deferred eviction as its own kernel (before calls that do not start with k_dd_fused)
__global__ void __launch_bounds__(256) k_evict_pending(Dev s, EvBuf b, P2P pm, int push) {
  evict_listed<8>(s, b, push ? &pm : nullptr, blockIdx.x, gridDim.x);
}

// Update (Alg. 3): block 0 plans this step's eviction (need, mode, LFU
// threshold T / K*, the bitmap blocks holding victims, R9) and
// publishes the plan; blocks 1..xb extract the victim keys once it is out;
// the other blocks do the ordered segment reduce + SGD + pending + clock.
// LFU bitmap plans end there: the victims are evicted by the first kernel of
// the next call (k_dd_fused / k_evict_pending) -- nothing reads or changes
// the cache in between, so the result is that of Evict() at the end of the
// update (R9).  The generic selection
// (LRU, LFU beyond the bitmaps, evict-all) and steps that rebuild the hash
// continue in this kernel after grid syncs.
__global__ void __launch_bounds__(UPD_THREADS)
k_update_fused(Dev s, Call c, const float* __restrict__ G, float lr, EvBuf b, int stage_rows, P2P pm, int push,
               int xb, int clock_only) {
  pdl_wait();
  const P2P* pp = push ? &pm : nullptr;
  extern __shared__ float4 dyn[];
  __shared__ uint32_t h[NBIN];
  __shared__ uint64_t bars[UPD_WARPS];
  __shared__ int dpop[LFU_CB_MAX];
  __shared__ unsigned s_dirty, s_ev, s_tomb;
  __shared__ int s_emode, s_rebuild, s_xlast;
  cg::grid_group grid = cg::this_grid();
  Ctl* ctl = s.ctl;
  dpop_init(dpop);
  if (threadIdx.x == 0) { s_dirty = 0; s_ev = 0; s_tomb = 0; }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { mbar_init(&bars[wid], 1); fence_mbar_init(); }
  TL_MIN(16);
  __syncthreads();
  const bool abort = ctl->abort;
  const int U = abort ? 0 : (c.rmode ? c.n : ctl->U);   // rmode: sorted positions, heads carry the work
  const uint32_t seq = ctl->lk_seq;   // set by the lookup; the plan flag carries it
  const int D4 = s.D >> 2;
  // wide rows (clock_only): k_seg_tma reduced the rows; this kernel steps the
  // clocks (after every slice read the dirty flag: the kernel boundary) and plans
  const bool xblock = blockIdx.x >= 1 && blockIdx.x <= xb;
  __shared__ Plan pl;
  if (blockIdx.x == 0 || xblock) {
    // ---- the eviction plan: block 0 publishes it for the other blocks'
    // end-of-kernel decision; the extraction blocks derive it themselves
    TL_MAX(22);
    make_plan(s, abort, &pl);
    TL_MAX(26);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->ncand = 0; ctl->nsub = 0; ctl->vmode = 0;
    ctl->need = pl.need;
    ctl->emode = pl.emode;
    ctl->rebuild_req = pl.rebuild;
    ctl->ev_ftop0 = (int32_t)pl.ftop;   // stable until the victims are freed
    ctl->T = pl.T;
    ctl->Kstar = pl.Kstar;
    ctl->needT = pl.needT;
    ctl->lowmask = pl.lowmask;
    ctl->generic = pl.emode == 2;
    __threadfence();
    st_release_u32(&ctl->plan_flag, seq);
    TL_MAX(23);
  }
  // the plan's mode as the other blocks read it (block 0's flag)
  auto read_plan = [&]() {
    if (threadIdx.x == 0) {
      if (blockIdx.x != 0)
        while (ld_acquire_u32(&ctl->plan_flag) != seq) __nanosleep(64);
      s_emode = abort ? 0 : __ldcg(&ctl->emode);
      s_rebuild = __ldcg(&ctl->rebuild_req);
    }
  };
  // blocks 1..xb: extract the victim keys (LFU bitmap path); ctl->nsel was
  // reset by this call's first kernel
  if (xblock) {
    if (threadIdx.x == 0) { s_emode = pl.emode; s_rebuild = pl.rebuild; }
    __syncthreads();
    TL_MAX(11);
    if (s_emode == 1) extract_victims(s, b, pl, (blockIdx.x - 1) * UPD_WARPS + wid, xb * UPD_WARPS, lane);
    TL_MAX(20);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_xlast = atomicAdd(&ctl->ext_blocks, 1) == xb - 1;
    __syncthreads();
    if (s_xlast && threadIdx.x == 0) {   // every victim key is listed
      ctl->ext_blocks = 0;
      const int nsel = __ldcg(&ctl->nsel);
      const bool defer = s_emode == 1 && !s_rebuild;
      ctl->nvict = s_emode == 1 ? nsel : 0;
      ctl->ev_nsel = nsel;
      ctl->ev_pending = (defer && nsel > 0) ? 1 : 0;
    }
  }
  // ---- the other blocks: ordered segment reduce + SGD + pending + clock, warp per unique key
  const int gw = blockIdx.x * UPD_WARPS + wid;
  const int nw = gridDim.x * UPD_WARPS;
  float4* mystg = dyn + (size_t)wid * (stage_rows + 1) * D4;
  uint32_t phase = 0;
  const float4* G4 = reinterpret_cast<const float4*>(G);
  const int rw = gw - (1 + xb) * UPD_WARPS, nrw = nw - (1 + xb) * UPD_WARPS;
  if (rw >= 0) {
    if (clock_only) {   // Cache.Clock, one lane per key
      for (int u = rw * 32 + lane; u < U; u += nrw * 32) {
        const int4 rec = __ldcg(&c.urec[u]);
        if (rec.x >= 0) s.cc[rec.x] = (uint32_t)rec.w + 1;
      }
    } else {
      for (int u = rw; u < U; u += nrw) segreduce_key(s, c, G4, lr, u, lane, mystg, &bars[wid], phase, stage_rows);
    }
  }
  TL_MAX(18);
  if (!xblock) read_plan();   // after this block's segment reduce (block 0: its own plan)
  __syncthreads();
  const int emode = s_emode;
  const bool rebuild = s_rebuild;
  // LFU bitmap plan (or nothing to evict), no hash rebuild, narrow rows: done
  // -- the victims wait for the next call's first kernel (uniform decision)
  if (emode != 2 && !rebuild) return;
  grid.sync();
  TL_MAX(19);
  // ---- in-kernel eviction: LFU bitmap victims (listed by blocks 1..xb)
  if (emode == 1) {
    const int nsel = __ldcg(&ctl->nsel);
    const int64_t ftop0 = __ldcg(&ctl->ev_ftop0);
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->ftop = (int32_t)(ftop0 + nsel);
    for (int i = gw; i < nsel; i += nw) {
      const int64_t key = __ldcg(&b.vsel[i]);
      uint64_t slot = 0;
      const int32_t e = warp_find_slot(s, key, lane, &slot);
      if (e >= 0) evict_entry(s, b, e, key, slot, lane, dpop, &s_dirty, &s_ev, &s_tomb, i, ftop0 + i, pp);
      else if (lane == 0) raise_err(ctl, 3 /*HET_ERR_PROTOCOL: a listed victim is not resident*/);
    }
  }
  // ---- generic selection (LRU, LFU fallback, evict-all) after all updates
  if (emode == 2) {
    generic_select(s, b, reinterpret_cast<uint64_t*>(dyn), h, grid);
    grid.sync();
    const int nv = ctl->nvict;
    const int64_t ftop0 = __ldcg(&ctl->ftop);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->ftop = (int32_t)(ftop0 + nv);
    for (int i = gw; i < nv; i += nw) {
      const int32_t e0 = b.victims[i];
      const int64_t key = s.ekey[e0];
      uint64_t slot = 0;
      int32_t e = warp_find_slot(s, key, lane, &slot);
      evict_entry(s, b, e, key, slot, lane, dpop, &s_dirty, &s_ev, &s_tomb, i, ftop0 + i, pp);
    }
  }
  TL_MAX(21);
  __syncthreads();
  dpop_flush(s, dpop);
  if (threadIdx.x == 0) {
    if (s_ev) atomicAdd(&s.cnt[C_EVICTIONS], (unsigned long long)s_ev);
    if (s_dirty) atomicAdd(&s.cnt[C_DIRTY_PUSHES], (unsigned long long)s_dirty);
    if (s_tomb) atomicAdd(&ctl->n_tomb, (int)s_tomb);
  }
  // ---- hash maintenance (rare): rebuild from the resident entries
  if (rebuild) {
    grid.sync();
    const int64_t HS = (int64_t)s.hmask + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HS; i += (int64_t)gridDim.x * blockDim.x)
      s.hslot[i] = HS_EMPTY;
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->n_tomb = 0; ctl->rebuild_req = 0; }
    for (int64_t e0 = (int64_t)gw * 32; e0 < s.Ecap; e0 += (int64_t)nw * 32) {
      int64_t e = e0 + lane;
      int64_t key = e < s.Ecap ? s.ekey[e] : -1;
      unsigned m = __ballot_sync(0xffffffffu, key >= 0);
      while (m) {
        int src = __ffs(m) - 1;
        int64_t k = __shfl_sync(0xffffffffu, key, src);
        warp_insert(s, k, (int32_t)(e0 + src), lane);
        m &= m - 1;
      }
    }
  }
}

// ------------------------------------------------------------------ K1 for 8192 < n <= 16384 (rmode)
// Eight CTAs rank every occurrence by a counting sort over 4096 key buckets
// (the top 12 bits of the key range: the keys are permuted ids, R15) and an
// exact rank inside each bucket: r(p) = offset(bucket) + #{q in the bucket:
// key_q < key_p, or key_q = key_p and q < p} -- the same stable sort as the
// rank count (R2), with n^2/4096 compares instead of n^2 (the Reddit-shaped
// batches: 14,208 distinct ids).  Extra blocks run the deferred eviction as
// in k_dd_fused.
constexpr int BK_THREADS = 1024, BK_BITS = 12, BK_N = 1 << BK_BITS, BK_MAX = 16384;
constexpr int BK_PF = 16;       // blocks issuing the lookup's L2 prefetches
constexpr int BK_CTAS = 8;      // CTAs that each build the bucket order and rank 1/8 of it
constexpr int EV_BLOCKS = 32;   // blocks of the deferred eviction beside the dedup
__global__ void __launch_bounds__(BK_THREADS)
k_dd_bucket(const int64_t* __restrict__ keys, int n, int pbits, Dev s, Call c, uint64_t t, int lookup, EvBuf eb,
            P2P pm, int push) {
  pdl_trigger();
  if ((int)blockIdx.x >= BK_CTAS + BK_PF) {
    evict_listed(s, eb, push ? &pm : nullptr, blockIdx.x - BK_CTAS - BK_PF, gridDim.x - BK_CTAS - BK_PF);
    return;
  }
  if ((int)blockIdx.x >= BK_CTAS) {   // the lookup's lines (hints), spread over BK_PF blocks
    if (!lookup) return;
    const int pb = blockIdx.x - BK_CTAS;
    for (int q = pb * BK_THREADS + threadIdx.x; q < n; q += BK_PF * BK_THREADS) {   // one pass
      const int64_t key = __ldg(&keys[q]);
      if (key < 0 || key >= s.R) continue;
      prefetch_l2(s.hslot + hash_home(s, key));
      prefetch_l2(s.hslot + hash_home(s, key) + 16);
      if (s.lfu_persist) prefetch_l2(s.count_by_key + key);
      if (key % s.world != s.rank) continue;
      const int64_t row = key / s.world;
      prefetch_l2(s.cg + row);
      for (uint32_t d = 0; d < s.D && d < 128; d += 32) prefetch_l2(s.W + row * s.D + d);
    }
    return;
  }
  TL_MIN(0);
  extern __shared__ __align__(16) uint32_t bk[];
  uint32_t* skey = bk;                 // [n]   the keys (32-bit)
  uint32_t* sord = bk + BK_MAX;        // [n]   positions grouped by bucket
  uint32_t* soff = bk + 2 * BK_MAX;    // [BK_N] bucket offsets
  uint32_t* scur = soff + BK_N;        // [BK_N] counts, then scatter cursors
  __shared__ int warp_sums[32];
  const int sh = max(0, s.kbits - BK_BITS);
  for (int b = threadIdx.x; b < BK_N; b += BK_THREADS) scur[b] = 0;
  __syncthreads();
  int bad = 0;
  {  // every key load of this thread in flight at once
    constexpr int IT = BK_MAX / BK_THREADS;
    int64_t kk[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int q = threadIdx.x + i * BK_THREADS;
      kk[i] = q < n ? __ldg(&keys[q]) : 0;
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) {
      const int q = threadIdx.x + i * BK_THREADS;
      if (q >= n) continue;
      if (kk[i] < 0 || kk[i] >= s.R) { bad = 1; continue; }
      skey[q] = (uint32_t)kk[i];
      atomicAdd(&scur[(uint32_t)kk[i] >> sh], 1u);
    }
  }
  bad = __syncthreads_or(bad);
  TL_X(4);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (lookup == 2) *c.pref_bad = bad;   // het_prefetch: the consuming lookup raises it
    else dd_begin(s, c, n, t, lookup, bad, 0);
  }
  if (bad) return;
  // exclusive scan of the bucket counts (4 per thread)
  {
    const int b0 = threadIdx.x * (BK_N / BK_THREADS);
    uint32_t v[BK_N / BK_THREADS];
    int sum = 0;
#pragma unroll
    for (int j = 0; j < BK_N / BK_THREADS; ++j) { v[j] = scur[b0 + j]; sum += v[j]; }
    int tot = 0;
    int ex = block_scan_int(sum, warp_sums, &tot);
#pragma unroll
    for (int j = 0; j < BK_N / BK_THREADS; ++j) { soff[b0 + j] = ex; scur[b0 + j] = ex; ex += v[j]; }
  }
  __syncthreads();
  TL_X(0);
  for (int q = threadIdx.x; q < n; q += BK_THREADS) sord[atomicAdd(&scur[skey[q] >> sh], 1u)] = q;
  __syncthreads();
  TL_X(1);
  // exact rank inside the bucket (scur now holds each bucket's end); CTA b
  // ranks positions [b per, (b+1) per) (the compare loops are shared-memory
  // bound: one CTA alone takes ~15 us at n = 14,208).  Every CTA built the
  // same buckets (in its own order inside a bucket, which the rank ignores).
  const int per = (n + BK_CTAS - 1) / BK_CTAS;
  const int q_lo = blockIdx.x * per, q_hi = min(n, q_lo + per);
  for (int q = q_lo + (int)threadIdx.x; q < q_hi; q += BK_THREADS) {
    const uint32_t k = skey[q], b = k >> sh;
    const uint32_t j0 = soff[b], j1 = scur[b];
    uint32_t r = j0;
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t qq = sord[j], kk = skey[qq];
      r += (kk < k) || (kk == k && (int)qq < q);
    }
    HET_ASSERT(r < (uint32_t)n);
    c.sortbuf0[r] = ((uint64_t)k << pbits) | (uint64_t)q;
    c.perm[r] = q;
  }
  TL_X(3);
}

// a lookup whose keys het_prefetch already deduplicated (NEXT-1):
// block 0 does the per-call begin (and raises a key outside [0, R) found by
// the prefetch), the other blocks the deferred eviction
__global__ void __launch_bounds__(256) k_begin_evict(Dev s, Call c, int n, uint64_t t, EvBuf eb, P2P pm, int push) {
  pdl_trigger();
  if (blockIdx.x > 0) {
    evict_listed<8>(s, eb, push ? &pm : nullptr, blockIdx.x - 1, gridDim.x - 1);
    return;
  }
  if (threadIdx.x == 0) dd_begin(s, c, n, t, 1, *c.pref_bad, 0);
}

int launch_begin_evict(const Dev& s, const Call& c, int n, uint64_t t, cudaStream_t st, void* evbuf,
                       const void* p2pview, bool evict) {
  P2P pm{};
  int push = 0;
  if (p2pview) { pm = *reinterpret_cast<const P2P*>(p2pview); push = 1; }
  k_begin_evict<<<1 + (evict ? 2 * EV_BLOCKS : 0), 256, 0, st>>>(s, c, n, t, *reinterpret_cast<EvBuf*>(evbuf), pm,
                                                                   push);
  return 1;
}

int launch_dd_bucket(const Dev& s, const Call& c, int n, int pbits, uint64_t t, int lookup, cudaStream_t st,
                     void* evbuf, const void* p2pview, bool evict) {
  const size_t smem = (2 * (size_t)BK_MAX + 2 * BK_N) * 4;   // keys, bucket order, offsets: 160 KB
  static uint64_t attr_devs = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_devs >> (dev & 63)) & 1)) {
    cudaFuncSetAttribute(k_dd_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_devs |= 1ull << (dev & 63);
  }
  P2P pm{};
  int push = 0;
  if (p2pview) { pm = *reinterpret_cast<const P2P*>(p2pview); push = 1; }
  k_dd_bucket<<<BK_CTAS + BK_PF + (evict ? EV_BLOCKS : 0), BK_THREADS, smem, st>>>(c.keys, n, pbits, s, c, t, lookup,
                                                                      *reinterpret_cast<EvBuf*>(evbuf), pm, push);
  return 1;
}

// ------------------------------------------------------------------ debug export of an rmode lookup
// One CTA: head flags of the sorted composites, a block scan for the unique
// index u of every head, then unique[u], seg_off[u], status[u] and the
// inverse by u -- the compact lookup log (R2) the rmode path never builds.
constexpr int CL_THREADS = 1024, CL_ITEMS = 16;   // n <= 16384 (the rmode dedups' bound)
__global__ void __launch_bounds__(CL_THREADS) k_compact_log(Dev s, Call c) {
  extern __shared__ int u_of[];   // [n]
  __shared__ int warp_sums[32];
  const int n = s.ctl->abort ? 0 : c.n, pb = c.pbits;
  const int i0 = threadIdx.x * CL_ITEMS;
  bool hd[CL_ITEMS];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < CL_ITEMS; ++k) {
    const int r = i0 + k;
    hd[k] = r < n && (r == 0 || (c.sortbuf0[r] >> pb) != (c.sortbuf0[r - 1] >> pb));
    cnt += hd[k];
  }
  int tot = 0;
  int u = block_scan_int(cnt, warp_sums, &tot);
#pragma unroll
  for (int k = 0; k < CL_ITEMS; ++k) {
    const int r = i0 + k;
    if (hd[k]) {
      u_of[r] = u;
      c.uniq[u] = (int64_t)(c.sortbuf0[r] >> pb);
      c.seg_off[u] = r;
      c.dbg_status[u] = c.status[r];
      ++u;
    }
  }
  if (threadIdx.x == 0) { c.seg_off[tot] = n; *c.dbg_U = tot; }
  __syncthreads();
  for (int pos = threadIdx.x; pos < n; pos += blockDim.x) c.dbg_inverse[pos] = u_of[c.inverse[pos]];
}

void launch_compact_log(const Dev& s, const Call& c, cudaStream_t st) {
  const size_t smem = (size_t)std::max(c.n, 1) * 4;
  cudaFuncSetAttribute(k_compact_log, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_compact_log<<<1, CL_THREADS, smem, st>>>(s, c);
}

// ------------------------------------------------------------------ launchers
constexpr int FUSED_MAX_DD_RANK = 8192;
constexpr int FUSED_MAX = 8192;

bool fused_ok(const Dev& s, int n) { return n <= FUSED_MAX; }


int launch_dd_fused(const Dev& s, const Call& c, int n, int pbits, uint64_t t, int lookup, cudaStream_t st,
                    void* evbuf, const void* p2pview, bool evict, int compact) {
  static uint64_t attr_devs = 0;   // devices whose function attribute is set
  int dev = 0;
  cudaGetDevice(&dev);
  if (!((attr_devs >> (dev & 63)) & 1)) {
    cudaFuncSetAttribute(k_dd_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, FUSED_MAX * 8);
    attr_devs |= 1ull << (dev & 63);
  }
  const int ndd = std::max(1, (n + 31) / 32);
  P2P pm{};
  int push = 0;
  if (p2pview) { pm = *reinterpret_cast<const P2P*>(p2pview); push = 1; }
  // wide rows: twice the eviction blocks (a warp per victim row of up to 16 KB)
  const int evb = evict ? (wide_rows(s.D) ? 2 * EV_BLOCKS : EV_BLOCKS) : 0;
  k_dd_fused<<<ndd + evb, DDF_THREADS, (size_t)std::max(n, 1) * 8, st>>>(
      c.keys, n, pbits, s, c, t, lookup, *reinterpret_cast<EvBuf*>(evbuf), pm, push, ndd, compact);
  return 1;
}

int launch_evict_pending(const Dev& s, void* evbuf, const void* p2pview, cudaStream_t st) {
  P2P pm{};
  int push = 0;
  if (p2pview) { pm = *reinterpret_cast<const P2P*>(p2pview); push = 1; }
  k_evict_pending<<<2 * EV_BLOCKS, 256, 0, st>>>(s, *reinterpret_cast<EvBuf*>(evbuf), pm, push);
  return 1;
}

// HET_PDL: 0 off, 1 dedup -> lookup, 2 also lookup -> cooperative update.
// Default: 2 at N = 1 (measured 31.75 -> 31.43 us per WDL step), 1 at N > 1
// (the update follows the cooperative exchange round there).
static int pdl_env() {
  static int m = -2;
  if (m == -2) {
    const char* e = getenv("HET_PDL");
    m = e ? atoi(e) : -1;
  }
  return m;
}
static int pdl_mode() { return pdl_env() >= 0 ? pdl_env() : 1; }
static bool pdl_update(const Dev& s) { return pdl_env() >= 0 ? pdl_env() >= 2 : s.world == 1; }

template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), int blocks, int threads, size_t smem, cudaStream_t st, bool pdl, bool coop,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (coop) {
    at[na].id = cudaLaunchAttributeCooperative;
    at[na].val.cooperative = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, k, args...);
}

int launch_lookup_fused(const Dev& s, const Call& c, float* out, cudaStream_t st, void* prof) {
  const int D4 = (int)s.D / 4;
  if (D4 >= 256 && D4 % 128 == 0) {            // wide rows
    if (c.rmode) {   // decisions (warp per key), then the row moves (per-thread copy pipelines)
      const int blocks = std::max(1, (c.n + LK_WARPS - 1) / LK_WARPS);
      void* pr = prof_begin(prof, "lookup_dec", st);
      launch_pdl(k_lookup_wide, blocks, LK_WARPS * 32, 0, st, pdl_mode() >= 1, false, s, c, out, 0);
      prof_end(prof, pr, st);
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      static bool attr = false;
      const size_t smem = (size_t)AS_MV[0] * AS_MV[1] * AS_T * 16;
      auto kern = k_mv_as<AS_MV[0], AS_MV[1]>;
      if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); attr = true; }
      const int S = D4 / (AS_T * AS_MV[1]);
      pr = prof_begin(prof, "lookup_mv", st);
      launch_pdl(kern, std::max(1, sms * AS_MV[2] / S) * S, AS_T, smem, st, pdl_mode() >= 1, false, s, c, out, 0,
                 (const float*)nullptr, (int64_t)0, (const int32_t*)nullptr);
      prof_end(prof, pr, st);
      return 2;
    }
    int G = 1;   // G warps per key (a power of two), decisions and moves in one kernel
    while (G * 2 <= std::min(LK_WARPS, D4 / 128)) G *= 2;
    const int blocks = std::max(1, (c.n + LK_WARPS / G - 1) / (LK_WARPS / G));
    void* pr = prof_begin(prof, "lookup_fused", st);
    launch_pdl(k_lookup_wide, blocks, LK_WARPS * 32, 0, st, pdl_mode() >= 1, false, s, c, out, G);
    prof_end(prof, pr, st);
    return 1;
  }
  int blocks = std::max(1, (c.n + LK_WARPS - 1) / LK_WARPS);
  const int agg = c.n > FUSED_MAX_DD_RANK;   // many misses: block-aggregated free-stack pops
  void* pr = prof_begin(prof, "lookup_fused", st);
  launch_pdl(k_lookup_fused, blocks, LK_WARPS * 32, 0, st, pdl_mode() >= 1, false, s, c, out, agg);
  prof_end(prof, pr, st);
  return 1;
}

int coop_sm_reserve() {
  static int r = -1;
  if (r < 0) {
    const char* e = getenv("HET_NCCL_CTAS");
    r = e ? std::max(1, atoi(e)) : 16;   // dense all-reduce blocks (peer memory or NCCL CTAs)
  }
  return r;
}

// cooperative launch configuration per (device, N > 1, D): the grid leaves
// coop_sm_reserve() SMs free at N > 1 and the staging depends on D
struct UpdCfg { int dev; bool multi; uint32_t D; int blocks; size_t smem; int stage_rows; };

int launch_scatter_wide(const Dev& s, const Call& c, float* out, cudaStream_t st, const float* resp, int64_t rec,
                        const int32_t* uslot) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static bool attr = false;
  const size_t smem = (size_t)AS_MV[0] * AS_MV[1] * AS_T * 16;
  auto kern = k_mv_as<AS_MV[0], AS_MV[1]>;
  if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); attr = true; }
  const int S = (int)(s.D / 4) / (AS_T * AS_MV[1]);
  kern<<<std::max(1, sms * AS_MV[2] / S) * S, AS_T, smem, st>>>(s, c, out, 1, resp, rec, uslot);
  return 1;
}

int launch_update_fused(const Dev& s, const Call& c, const float* grads, float lr, void* evbuf, cudaStream_t st,
                        const void* p2pview, void* prof) {
  static std::vector<UpdCfg> cfgs;
  int dev = 0;
  cudaGetDevice(&dev);
  const bool multi = s.world > 1;
  const UpdCfg* cf = nullptr;
  for (const UpdCfg& x : cfgs)
    if (x.dev == dev && x.multi == multi && x.D == s.D) cf = &x;
  if (!cf) {
    UpdCfg x{dev, multi, s.D, 0, 0, 0};
    const int rowbytes = (int)s.D * 4;
    x.stage_rows = std::min(32, 12288 / rowbytes);
    if (x.stage_rows < 4) x.stage_rows = 0;
    size_t stg = x.stage_rows ? (size_t)UPD_WARPS * (x.stage_rows + 1) * rowbytes : 0;
    x.smem = std::max(stg, (size_t)SUBMAX * 8);
    cudaFuncSetAttribute(k_update_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)x.smem);
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_update_fused, UPD_THREADS, x.smem);
    // N > 1: leave NCCL's SMs free (the overlapped dense all-reduce)
    x.blocks = (multi ? sms - coop_sm_reserve() : sms) * std::max(per, 1);
    cfgs.push_back(x);
    cf = &cfgs.back();
  }
  const int coop_blocks = cf->blocks;
  const size_t smem = cf->smem;
  const int stage_rows = cf->stage_rows;
  EvBuf& b = *reinterpret_cast<EvBuf*>(evbuf);
  Dev sd = s;
  Call cd = c;
  int sr = stage_rows;
  P2P pm{};
  int push = 0;
  if (p2pview) { pm = *reinterpret_cast<const P2P*>(p2pview); push = 1; }
  int xb = std::max(1, std::min(8, coop_blocks / 16));   // extraction blocks (after block 0's plan)
  static const int xb_env = getenv("HET_XB") ? atoi(getenv("HET_XB")) : 0;   // measurement override
  if (xb_env > 0) xb = std::min(xb_env, coop_blocks - 2);
  const int D4 = (int)s.D / 4;
  int clock_only = (D4 >= 256 && D4 % 128 == 0) ? 1 : 0;   // wide rows: k_seg_as reduces the rows first
  int launches = 1;
  if (clock_only) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cf->dev);
    static bool attr = false;
    const size_t ssm = (size_t)AS_SEG[0] * AS_SEG[1] * AS_T * 16;
    auto kern = k_seg_as<AS_SEG[0], AS_SEG[1], AS_SEG[2]>;
    if (!attr) { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm); attr = true; }
    const int S = D4 / (AS_T * AS_SEG[1]);
    void* pr = prof_begin(prof, "seg_wide", st);
    launch_pdl(kern, std::max(1, sms * AS_SEG[3] / S) * S, AS_T, ssm, st, pdl_mode() >= 1, false, sd, cd, grads, lr);
    prof_end(prof, pr, st);
    launches += 1;
  }
  void* args[] = {(void*)&sd, (void*)&cd, (void*)&grads, (void*)&lr, (void*)&b, (void*)&sr, (void*)&pm, (void*)&push,
                  (void*)&xb, (void*)&clock_only};
  void* pr = prof_begin(prof, "update_fused", st);
  if (pdl_update(s))
    launch_pdl(k_update_fused, coop_blocks, UPD_THREADS, smem, st, true, true, sd, cd, grads, lr, b, sr, pm, push, xb,
               clock_only);
  else
    cudaLaunchCooperativeKernel((void*)k_update_fused, dim3(coop_blocks), dim3(UPD_THREADS), args, smem, st);
  prof_end(prof, pr, st);
  return launches;
}

}  // namespace het
