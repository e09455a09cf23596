// K1 dedup in ONE CTA: stable LSD radix sort of (key, position) pairs over
// the key's kbits bits (CUB's BlockRadixSort inside our own kernel), then
// segment heads, unique/inverse/perm/seg_off and the per-call begin, all
// without leaving the block (no second kernel, no last-block hand-off).
//
//   Alg. 1 line 5 "unique key set"; R2: unique keys ascending,
//   inverse int32 into unique, perm = positions grouped by key in ascending
//   position (the sort is stable, input in position order).
//
// 1024 threads x ITEMS keys (ITEMS = 4, 8, 16: n <= 4096, 8192, 16384).
// Padding items carry positions >= n; a real key equal to the padding key
// still sorts before them (stability), and they are never heads.
#include <cub/block/block_radix_sort.cuh>

#include "het_internal.cuh"

namespace het {

constexpr int DR_THREADS = 1024;

template <int ITEMS>
__global__ void __launch_bounds__(DR_THREADS)
k_dd_radix(const int64_t* __restrict__ keys, int n, int kbits, Dev s, Call c, uint64_t t, int lookup) {
  using BRS = cub::BlockRadixSort<uint32_t, DR_THREADS, ITEMS, int32_t>;
  extern __shared__ __align__(16) unsigned char dr_smem[];
  auto& tmp = *reinterpret_cast<typename BRS::TempStorage*>(dr_smem);
  __shared__ uint32_t s_last_key[DR_THREADS / 32];
  __shared__ int warp_sums[32];
  __shared__ int s_bad;
  Ctl* ctl = s.ctl;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  uint32_t k[ITEMS];
  int32_t p[ITEMS];
  int bad = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {             // blocked: thread t holds positions t*ITEMS + i
    const int q = threadIdx.x * ITEMS + i;
    int64_t kk = q < n ? __ldg(&keys[q]) : 0;
    if (q < n && (kk < 0 || kk >= s.R)) bad = 1;
    k[i] = q < n ? (uint32_t)kk : 0xFFFFFFFFu;
    p[i] = q;
  }
  if (bad) s_bad = 1;
  if (threadIdx.x == 0) {                        // per-call begin
    if (lookup) {
      if (t == CLOCK_AUTO) { t = ctl->t_auto; ctl->t_auto = t + 1; }
      ctl->t_cur = t;
      ctl->lk_seq = ctl->lk_seq + 1;
      s.cnt[C_LOOKUPS] += 1;
      s.cnt[C_KEYS] += (unsigned long long)n;
    }
    ctl->abort = 0;
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) { raise_err(ctl, 2 /*HET_ERR_KEY_RANGE*/); ctl->U = 0; c.seg_off[0] = 0; }
    return;
  }
  BRS(tmp).Sort(k, p, 0, kbits < 32 ? kbits + 1 : 32);   // +1 bit: the padding key sorts last
  // ---- heads: key differs from the previous sorted item (blocked layout)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t prev = __shfl_up_sync(0xffffffffu, k[ITEMS - 1], 1);
  if (lane == 31) s_last_key[wid] = k[ITEMS - 1];
  __syncthreads();
  if (lane == 0) prev = wid ? s_last_key[wid - 1] : 0u;
  unsigned hm = 0;
  int cnt = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = threadIdx.x * ITEMS + i;
    const bool valid = p[i] < n;
    const bool head = valid && (j == 0 || k[i] != (i ? k[i - 1] : prev));
    if (head) { hm |= 1u << i; ++cnt; }
  }
  // block exclusive scan of the head counts
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) warp_sums[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  const int U = warp_sums[31];
  int u = (wid ? warp_sums[wid - 1] : 0) + v - cnt - 1;   // unique index of the last head seen
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int j = threadIdx.x * ITEMS + i;
    if (p[i] < n) {
      if ((hm >> i) & 1u) {
        ++u;
        c.uniq[u] = (int64_t)k[i];
        c.seg_off[u] = j;
      }
      c.perm[j] = p[i];
      c.inverse[p[i]] = u;
    }
  }
  if (threadIdx.x == 0) { c.seg_off[U] = n; ctl->U = U; }
}

template <int ITEMS>
static size_t dr_smem() {
  return sizeof(typename cub::BlockRadixSort<uint32_t, DR_THREADS, ITEMS, int32_t>::TempStorage);
}

bool dd_radix_ok(int n) { return n <= DR_THREADS * 16; }

int launch_dd_radix(const Dev& s, const Call& c, int n, uint64_t t, int lookup, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dd_radix<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dr_smem<4>());
    cudaFuncSetAttribute(k_dd_radix<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dr_smem<8>());
    cudaFuncSetAttribute(k_dd_radix<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dr_smem<16>());
    attr = true;
  }
  const int kb = s.kbits;
  if (n <= DR_THREADS * 4)
    k_dd_radix<4><<<1, DR_THREADS, dr_smem<4>(), st>>>(c.keys, n, kb, s, c, t, lookup);
  else if (n <= DR_THREADS * 8)
    k_dd_radix<8><<<1, DR_THREADS, dr_smem<8>(), st>>>(c.keys, n, kb, s, c, t, lookup);
  else
    k_dd_radix<16><<<1, DR_THREADS, dr_smem<16>(), st>>>(c.keys, n, kb, s, c, t, lookup);
  return 1;
}

}  // namespace het
