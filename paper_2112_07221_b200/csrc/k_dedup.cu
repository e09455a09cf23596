// K1 dedup: the "unique embedding key set" of a mini-batch (Alg. 1 line 5,
// PAPER.md:462; §4.2 "remove the duplicate keys") with the inverse
// index and the stable grouping of positions by key (reading R2: unique keys
// ascending, positions ascending within a key).
//
// Design: every occurrence becomes one 64-bit composite (key << pbits) | pos;
// composites are distinct, so sorting them is a stable sort of (key, pos).
//  * n <= 16384: one CTA sorts all composites in shared memory (bitonic),
//    flags segment heads, block-scans them and writes unique/inverse/perm/
//    seg_off in the same kernel (one launch).
//  * larger n: CTA-tile bitonic sorts of 8192 composites, log2(n/8192) merge
//    passes (each element finds its rank in the partner run by binary
//    search), then a three-kernel reduce/scan/write for the outputs.
#include <cooperative_groups.h>

#include <algorithm>

#include "het_internal.cuh"

namespace cg = cooperative_groups;

namespace het {

constexpr int DD_THREADS = 1024;
constexpr int DD_SMALL_MAX = 16384;   // 128 KB of composites in smem
constexpr int TILE = 8192;            // large-path CTA tile

__device__ __forceinline__ void bitonic_smem(uint64_t* a, int npad) {
  for (int k = 2; k <= npad; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < (npad >> 1); i += blockDim.x) {
        int lo = 2 * j * (i / j) + (i % j);
        int hi = lo + j;
        bool up = (lo & k) == 0;
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
      }
      __syncthreads();
    }
  }
}

// exclusive block scan of one int per thread; returns the exclusive prefix, total in *tot
__device__ __forceinline__ int block_excl_scan(int x, int* warp_sums, int* tot) {
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
    if (lane < nw) warp_sums[lane] = w;       // inclusive
  }
  __syncthreads();
  int base = wid ? warp_sums[wid - 1] : 0;
  *tot = warp_sums[nw - 1];
  __syncthreads();
  return base + v - x;
}

// Cluster dedup for n <= 16384: the padded composite array is split over a
// thread-block cluster of CS CTAs (CS = npad / (1024 E), up to 8); thread t of
// CTA r holds elements [r*chunk + t*E, ... + E) in registers.  Bitonic stages
// with partner distance j < E run inside a thread, E <= j < 32E through warp
// shuffles, 32E <= j < chunk through shared memory, and j >= chunk through
// distributed shared memory (the partner CTA's buffer, cluster.sync per
// stage).  Buffers alternate between stages so one barrier per stage suffices.
// Segment heads are block-scanned per CTA and offset by the totals of the
// lower-ranked CTAs read over DSMEM.
template <int E>
__global__ void __launch_bounds__(DD_THREADS, 1)
k_dedup_cluster(const int64_t* __restrict__ keys, int n, int npad, int64_t R, int pbits, Ctl* ctl,
                int64_t* uniq, int32_t* inverse, int32_t* perm, int32_t* seg_off) {
  extern __shared__ uint64_t sm[];              // [2][chunk]
  __shared__ int warp_sums[32];
  __shared__ uint64_t warp_last[32];
  __shared__ int s_flag, s_total;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  const int csize = (int)cl.num_blocks();
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int chunk = blockDim.x * E;
  const int gbase = crank * chunk;
  uint64_t r[E];
  int bad = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    int j = gbase + tid * E + q;
    uint64_t c = ~0ull;
    if (j < n) {
      int64_t k = keys[j];
      if (k < 0 || k >= R) bad = 1;
      c = ((uint64_t)k << pbits) | (uint64_t)j;
    }
    r[q] = c;
  }
  bad = __syncthreads_or(bad);
  if (tid == 0) s_flag = bad;
  cl.sync();
  int anybad = 0;
  for (int q = 0; q < csize; ++q) anybad |= *cl.map_shared_rank(&s_flag, q);
  if (anybad) {
    if (crank == 0 && tid == 0) { raise_err(ctl, 2 /*HET_ERR_KEY_RANGE*/); ctl->U = 0; seg_off[0] = 0; }
    cl.sync();
    return;
  }
  int pb = 0;
  for (int k = 2; k <= npad; k <<= 1) {
    int j = k >> 1;
    if (j >= chunk) {                               // cross-CTA stages (DSMEM)
      for (; j >= chunk; j >>= 1) {
        uint64_t* buf = sm + pb * chunk;
#pragma unroll
        for (int q = 0; q < E; ++q) buf[tid * E + q] = r[q];
        cl.sync();
        int pr = crank ^ (j / chunk);
        const uint64_t* rb = cl.map_shared_rank(buf, pr);
        bool lower = (crank & (j / chunk)) == 0;
#pragma unroll
        for (int q = 0; q < E; ++q) {
          uint64_t x = r[q], y = rb[tid * E + q];
          bool up = (((gbase + tid * E + q) & k) == 0);
          r[q] = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
        }
        pb ^= 1;
      }
      cl.sync();                                    // remote reads done before buffers are reused
    }
    if (j >= 32 * E) {                              // intra-CTA shared-memory stages
      for (; j >= 32 * E; j >>= 1) {
        uint64_t* buf = sm + pb * chunk;
#pragma unroll
        for (int q = 0; q < E; ++q) buf[tid * E + q] = r[q];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < E; ++q) {
          int li = tid * E + q;
          uint64_t x = r[q], y = buf[li ^ j];
          bool lower = (li & j) == 0;
          bool up = (((gbase + li) & k) == 0);
          r[q] = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
        }
        pb ^= 1;
      }
    }
    for (; j >= E; j >>= 1) {                       // warp shuffles
      int lm = j / E;
      bool lower = (tid & lm) == 0;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        uint64_t x = r[q];
        uint64_t y = __shfl_xor_sync(0xffffffffu, x, lm);
        bool up = (((gbase + tid * E + q) & k) == 0);
        r[q] = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
      }
    }
#pragma unroll
    for (int jj = E / 2; jj > 0; jj >>= 1) {         // inside the thread
      if (jj > (k >> 1)) continue;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if ((q & jj) == 0) {
          bool up = (((gbase + tid * E + q) & k) == 0);
          uint64_t x = r[q], y = r[q + jj];
          if ((x > y) == up) { r[q] = y; r[q + jj] = x; }
        }
      }
    }
  }
  // previous element of each thread's first element (previous thread / warp / CTA)
  uint64_t prev = __shfl_up_sync(0xffffffffu, r[E - 1], 1);
  if (lane == 31) warp_last[tid >> 5] = r[E - 1];
  __syncthreads();
  if (tid == 0) s_total = 0;
  cl.sync();
  if (lane == 0) {
    if (tid >> 5) prev = warp_last[(tid >> 5) - 1];
    else prev = crank ? cl.map_shared_rank(warp_last, crank - 1)[(blockDim.x >> 5) - 1] : ~0ull;
  }
  int heads = 0;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    int jg = gbase + tid * E + q;
    uint64_t p = q ? r[q - 1] : prev;
    if (jg < n && (jg == 0 || (r[q] >> pbits) != (p >> pbits))) ++heads;
  }
  int tot;
  int u = block_excl_scan(heads, warp_sums, &tot);
  if (tid == 0) s_total = tot;
  cl.sync();
  int base = 0, all = 0;
  for (int q = 0; q < csize; ++q) {
    int tq = *cl.map_shared_rank(&s_total, q);
    if (q < crank) base += tq;
    all += tq;
  }
  u += base - 1;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    int jg = gbase + tid * E + q;
    if (jg < n) {
      uint64_t c = r[q];
      uint64_t p = q ? r[q - 1] : prev;
      int pos = (int)(c & ((1ull << pbits) - 1));
      if (jg == 0 || (c >> pbits) != (p >> pbits)) {
        ++u;
        uniq[u] = (int64_t)(c >> pbits);
        seg_off[u] = jg;
      }
      perm[jg] = pos;
      inverse[pos] = u;
    }
  }
  if (crank == 0 && tid == 0) { seg_off[all] = n; ctl->U = all; }
  cl.sync();   // keep every CTA's shared memory alive until remote reads finish
}

// ------------------------------------------------------------- rank path
// n <= RANK_MAX: the stable-sort position of occurrence p is the number of
// composites smaller than its own, counted by brute force over the whole GPU
// (n^2 compares with no synchronisation: every block stages all composites
// in shared memory, its 32-lane tile of elements is compared against a 1/16
// share of them per warp).  A second, single-CTA kernel flags segment heads,
// block-scans them and writes unique/inverse/perm/seg_off.
constexpr int RANK_MAX = 8192;
constexpr int RANK_WARPS = 16;

__global__ void __launch_bounds__(RANK_WARPS * 32)
k_rank_sort(const int64_t* __restrict__ keys, int n, int64_t R, int pbits, Ctl* ctl, uint64_t* sorted) {
  extern __shared__ uint64_t comp[];
  __shared__ int part[RANK_WARPS][32];
  int bad = 0;
  constexpr int RI = RANK_MAX / (RANK_WARPS * 32);
  {  // all key loads of this thread in flight at once
    int64_t kk[RI];
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      const int q = threadIdx.x + i * RANK_WARPS * 32;
      kk[i] = q < n ? __ldg(&keys[q]) : 0;
    }
#pragma unroll
    for (int i = 0; i < RI; ++i) {
      const int q = threadIdx.x + i * RANK_WARPS * 32;
      if (q < n) {
        if (kk[i] < 0 || kk[i] >= R) bad = 1;
        comp[q] = ((uint64_t)kk[i] << pbits) | (uint64_t)q;
      }
    }
  }
  if (__syncthreads_or(bad)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_err(ctl, 2 /*HET_ERR_KEY_RANGE*/);
    return;
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  const uint64_t mine = p < n ? comp[p] : ~0ull;
  const int per = (n + RANK_WARPS - 1) / RANK_WARPS;
  const int q0 = wid * per, q1 = min(n, q0 + per);
  int cnt = 0;
#pragma unroll 8
  for (int q = q0; q < q1; ++q) cnt += comp[q] < mine;   // broadcast read
  part[wid][lane] = cnt;
  __syncthreads();
  if (wid == 0 && p < n) {
    int r = 0;
#pragma unroll
    for (int w = 0; w < RANK_WARPS; ++w) r += part[w][lane];
    sorted[r] = mine;
  }
}

__global__ void __launch_bounds__(DD_THREADS)
k_dedup_finish(const uint64_t* __restrict__ sorted, int n, int pbits, Ctl* ctl, int64_t* uniq,
               int32_t* inverse, int32_t* perm, int32_t* seg_off) {
  __shared__ int warp_sums[32];
  if (ctl->abort) {
    if (threadIdx.x == 0) { ctl->U = 0; seg_off[0] = 0; }
    return;
  }
  const int items = (n + blockDim.x - 1) / blockDim.x;
  const int j0 = threadIdx.x * items;
  int heads = 0;
  uint64_t prev = j0 > 0 && j0 < n ? sorted[j0 - 1] : ~0ull;
  for (int i = 0; i < items; ++i) {
    int j = j0 + i;
    if (j >= n) break;
    uint64_t c = sorted[j];
    if (j == 0 || (c >> pbits) != (prev >> pbits)) ++heads;
    prev = c;
  }
  int tot;
  int u = block_excl_scan(heads, warp_sums, &tot) - 1;
  prev = j0 > 0 && j0 < n ? sorted[j0 - 1] : ~0ull;
  for (int i = 0; i < items; ++i) {
    int j = j0 + i;
    if (j >= n) break;
    uint64_t c = sorted[j];
    int pos = (int)(c & ((1ull << pbits) - 1));
    if (j == 0 || (c >> pbits) != (prev >> pbits)) {
      ++u;
      uniq[u] = (int64_t)(c >> pbits);
      seg_off[u] = j;
    }
    perm[j] = pos;
    inverse[pos] = u;
    prev = c;
  }
  if (threadIdx.x == 0) { seg_off[tot] = n; ctl->U = tot; }
}

// ------------------------------------------------------------- large path
__global__ void __launch_bounds__(DD_THREADS)
k_tile_sort(const int64_t* __restrict__ keys, int n, int64_t R, int pbits, Ctl* ctl, uint64_t* out) {
  extern __shared__ uint64_t sm[];
  int base = blockIdx.x * TILE;
  int len = min(TILE, n - base);
  int bad = 0;
  for (int j = threadIdx.x; j < TILE; j += blockDim.x) {
    uint64_t c = ~0ull;
    if (j < len) {
      int64_t k = keys[base + j];
      if (k < 0 || k >= R) bad = 1;
      c = ((uint64_t)k << pbits) | (uint64_t)(base + j);
    }
    sm[j] = c;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) raise_err(ctl, 2);
  bitonic_smem(sm, TILE);
  for (int j = threadIdx.x; j < len; j += blockDim.x) out[base + j] = sm[j];
}

// merge sorted runs of length `width` pairwise: src -> dst
__global__ void k_merge(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, int n, int width) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int run = i / width;
  int a0 = (run & ~1) * width;
  int mid = min(a0 + width, n);
  int b1 = min(a0 + 2 * width, n);
  uint64_t x = src[i];
  int lo, hi;
  if (i < mid) { lo = mid; hi = b1; }   // element of A: count B elements < x
  else { lo = a0; hi = mid; }           // element of B: count A elements < x
  int l = lo, h = hi;
  while (l < h) {
    int m = (l + h) >> 1;
    if (src[m] < x) l = m + 1; else h = m;
  }
  int rank = l - lo;
  int out = (i < mid) ? (i - a0) + rank + a0 : (i - mid) + rank + a0;
  dst[out] = x;
}

constexpr int SCAN_BLK = 1024;

__global__ void k_head_count(const uint64_t* __restrict__ c, int n, int pbits, int32_t* blockcnt) {
  __shared__ int warp_sums[32];
  int j = blockIdx.x * SCAN_BLK + threadIdx.x;
  int h = (j < n && (j == 0 || (c[j] >> pbits) != (c[j - 1] >> pbits))) ? 1 : 0;
  int tot;
  block_excl_scan(h, warp_sums, &tot);
  if (threadIdx.x == 0) blockcnt[blockIdx.x] = tot;
}

__global__ void k_scan_blocks(int32_t* blockcnt, int nb, Ctl* ctl) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    int b = b0 + threadIdx.x;
    int x = b < nb ? blockcnt[b] : 0;
    int tot;
    int ex = block_excl_scan(x, warp_sums, &tot);
    if (b < nb) blockcnt[b] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->U = carry;
}

__global__ void k_head_write(const uint64_t* __restrict__ c, int n, int pbits, const int32_t* blockoff,
                             Ctl* ctl, int64_t* uniq, int32_t* inverse, int32_t* perm, int32_t* seg_off) {
  __shared__ int warp_sums[32];
  int j = blockIdx.x * SCAN_BLK + threadIdx.x;
  uint64_t x = j < n ? c[j] : 0;
  int h = (j < n && (j == 0 || (x >> pbits) != (c[j - 1] >> pbits))) ? 1 : 0;
  int tot;
  int ex = block_excl_scan(h, warp_sums, &tot);
  if (j < n) {
    int u = blockoff[blockIdx.x] + ex + h - 1;
    int pos = (int)(x & ((1ull << pbits) - 1));
    if (h) { uniq[u] = (int64_t)(x >> pbits); seg_off[u] = j; }
    perm[j] = pos;
    inverse[pos] = u;
  }
  if (j == n - 1) seg_off[ctl->U] = n;
}

__global__ void k_abort_if_bad(Ctl* ctl, int32_t* seg_off) {
  if (ctl->abort) { ctl->U = 0; seg_off[0] = 0; }
}

int launch_dedup(const Call& c, int n, int64_t R, int pbits, Ctl* ctl, cudaStream_t st) {
  if (n <= RANK_MAX) {
    int blocks = std::max(1, (n + 31) / 32);
    k_rank_sort<<<blocks, RANK_WARPS * 32, (size_t)std::max(n, 1) * 8, st>>>(c.keys, n, R, pbits, ctl, c.sortbuf0);
    k_dedup_finish<<<1, DD_THREADS, 0, st>>>(c.sortbuf0, n, pbits, ctl, c.uniq, c.inverse, c.perm, c.seg_off);
    return 2;
  }
  if (n <= DD_SMALL_MAX) {
    int npad = 32;
    while (npad < n) npad <<= 1;
    int E = npad <= 8192 ? 1 : npad / 8192;          // elements per thread
    int threads = std::min(npad / E, DD_THREADS);
    int csize = npad / (threads * E);                  // CTAs in the cluster (1..8)
    size_t smem = (size_t)2 * threads * E * 8;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (E == 1)
      cudaLaunchKernelEx(&cfg, k_dedup_cluster<1>, c.keys, n, npad, R, pbits, ctl, c.uniq, c.inverse, c.perm, c.seg_off);
    else
      cudaLaunchKernelEx(&cfg, k_dedup_cluster<2>, c.keys, n, npad, R, pbits, ctl, c.uniq, c.inverse, c.perm, c.seg_off);
    return 1;
  }
  int launches = 0;
  int ntiles = (n + TILE - 1) / TILE;
  k_tile_sort<<<ntiles, DD_THREADS, TILE * 8, st>>>(c.keys, n, R, pbits, ctl, c.sortbuf0);
  ++launches;
  uint64_t* a = c.sortbuf0;
  uint64_t* b = c.sortbuf1;
  for (int w = TILE; w < n; w <<= 1) {
    k_merge<<<(n + 255) / 256, 256, 0, st>>>(a, b, n, w);
    ++launches;
    uint64_t* t = a; a = b; b = t;
  }
  int nb = (n + SCAN_BLK - 1) / SCAN_BLK;
  k_head_count<<<nb, SCAN_BLK, 0, st>>>(a, n, pbits, c.blockbuf);
  k_scan_blocks<<<1, 1024, 0, st>>>(c.blockbuf, nb, ctl);
  k_head_write<<<nb, SCAN_BLK, 0, st>>>(a, n, pbits, c.blockbuf, ctl, c.uniq, c.inverse, c.perm,
                                        c.seg_off);
  k_abort_if_bad<<<1, 1, 0, st>>>(ctl, c.seg_off);
  return launches + 4;
}

void dedup_set_attrs() {
  cudaFuncSetAttribute(k_rank_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, RANK_MAX * 8);
  cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 8);
}

}  // namespace het
