// K7 segment reduce + SGD apply + clock for the per-phase path (large batches).
//
//   Cache.Update + Cache.Clock: for every unique key u
//   acc = +0.0f, then + G[pos] for its occurrences in ascending batch position
//   (R11), delta = (-lr) * acc, v += delta, p = (dirty ? p : +0) + delta (R13),
//   c_c += 1.  fp32 round-to-nearest adds and multiplies, no contraction (R17).
//
// The order of the sum is fixed per column, so a key's occurrences are a
// dependent chain of adds that the method cannot reassociate.  In the
// Criteo-shaped workload (Zipf 0.7 over fields with as few as 3 values) keys
// with more than 32 occurrences are <1 % of the unique keys but ~50 % of the
// rows at batch 32768; the heaviest key has ~16K occurrences (8 MB of rows).
// Measured on B200 (tools/ring_bench.cu, the timeline build): one SM ingests
// at most ~50 GB/s whatever the mechanism (cp.async rows, per-row bulk
// copies, contiguous 16 KB bulk copies), per-row cp.async.bulk issues at ~60
// cycles a copy, and 128 B cp.async slices of scattered rows are issue-bound
// at ~16 GB/s per SM.  So a heavy key must be spread over many SMs by columns,
// and column slices must be moved as tiles, not rows:
//
//   k_heavy_list  lists heavy keys by power-of-two size class, snapshots their
//                 dirty flag and takes their clock step (slices run on
//                 different SMs).
//   k_heavy_gather  (side stream) copies every heavy occurrence row into
//                 the slice-major hbuf[slice][j][16] = G[perm[j]][slice] -- all
//                 SMs, warp per row, coalesced -- so each (key, slice) is one
//                 contiguous block.  (A 2D TMA tile over a row-major copy was
//                 tried first: 64 B box rows cost the TMA unit ~15 cycles each.)
//   k_sr_heavy    (side stream, highest priority) items = (heavy key,
//                 16-column slice); two pipelines per SM, each an elected
//                 producer issuing one contiguous bulk copy (up to 256 rows x
//                 64 B = 16 KB) per stage from hbuf into a 4-stage ring, and a
//                 consumer warp adding in ascending
//                 position, one lane per column, writing the slice's sums
//                 over the item's first hbuf row.  Items are dealt largest
//                 size class first, in snake order over the pipelines.
//   k_heavy_apply (side stream) SGD + pending for the heavy keys.
//   k_sr_light    (main stream, concurrently) keys with <= SR_HEAVY
//                 occurrences: a 16-lane half-warp per key, up to 4 occurrence
//                 rows in flight per lane, v/p loaded alongside.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "het_internal.cuh"

namespace het {

constexpr int SR_HEAVY = 32;        // occurrences above which a key goes to k_sr_heavy
constexpr int HV_CTAS = 148;        // one heavy CTA per SM (light blocks co-reside)
constexpr int HV_PIPES = 2;         // pipelines per CTA: (producer warp, consumer warp, ring)
constexpr int HV_STAGES = 4;
constexpr int HV_BR = 256;          // rows per stage (TMA box rows)
constexpr int HV_W = 16;            // columns per slice (TMA box columns, 64 B)
constexpr int LT_THREADS = 256;

__device__ __forceinline__ float4 f4add_s(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float4 f4scale_s(float a, float4 b) {
  return make_float4(__fmul_rn(a, b.x), __fmul_rn(a, b.y), __fmul_rn(a, b.z), __fmul_rn(a, b.w));
}

// ------------------------------------------------------------------ heavy list
// Lists the heavy keys by size bucket b = floor(log2(count)) (bucket b holds
// at most cap >> b keys, placed at offset bucket_off(b)) and takes their
// Cache.Clock step here: a heavy key's column slices run on different SMs, so
// the dirty flag (c_c > c_s before the update, R13) is snapshotted into the
// list entry (bit 31) and c_c advanced once, before any slice starts.
__host__ __device__ __forceinline__ int bucket_off(int b, int cap) {
  int off = 0;
  for (int q = 5; q < b; ++q) off += (cap >> q) + 1;
  return off;
}
__global__ void k_heavy_list(Dev s, Call c, int cap) {
  Ctl* ctl = s.ctl;
  if (ctl->abort) return;
  const int U = ctl->U;
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < U; u += gridDim.x * blockDim.x) {
    const int cnt = c.seg_off[u + 1] - c.seg_off[u];
    if (cnt > SR_HEAVY) {
      const int32_t e = c.uentry[u];
      const uint32_t ecc = s.cc[e];
      const int32_t ent = u | (ecc > s.cs[e] ? (int32_t)0x80000000 : 0);
      s.cc[e] = ecc + 1;   // Cache.Clock
      const int b = 31 - __clz(cnt);   // >= 5
      c.hlist[bucket_off(b, cap) + atomicAdd(&ctl->nbucket[b], 1)] = ent;
    }
  }
}

// ------------------------------------------------------------------ light keys
__global__ void __launch_bounds__(LT_THREADS)
k_sr_light(Dev s, Call c, const float* __restrict__ G, float lr, int heavy) {
  Ctl* ctl = s.ctl;
  const int lane = threadIdx.x & 31, half = lane >> 4, hl = lane & 15;
  const unsigned hm = 0xFFFFu << (half * 16);
  const int u = (blockIdx.x * LT_THREADS + threadIdx.x) >> 4;
  if (ctl->abort || u >= ctl->U) return;
  const int j0 = c.seg_off[u], cnt = c.seg_off[u + 1] - j0;
  if (cnt > heavy) return;
  const int32_t e = c.uentry[u];
  const int pos0 = hl < cnt ? __ldg(&c.perm[j0 + hl]) : 0;
  const uint32_t ecc = s.cc[e], ecs = s.cs[e];
  const bool dirty = ecc > ecs;
  const int D4 = s.D >> 2;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* G4 = reinterpret_cast<const float4*>(G);
  float4* vr = reinterpret_cast<float4*>(s.v + (int64_t)e * s.D);
  float4* pr = reinterpret_cast<float4*>(s.p + (int64_t)e * s.D);
  const float nlr = -lr;
  for (int d0 = 0; d0 < D4; d0 += 32) {
    const int da = d0 + hl, db = d0 + 16 + hl;
    const bool aa = da < D4, ab = db < D4;
    const float4 va = aa ? vr[da] : zero, vb = ab ? vr[db] : zero;
    const float4 pa = (aa && dirty) ? pr[da] : zero, pb = (ab && dirty) ? pr[db] : zero;
    float4 acc0 = zero, acc1 = zero;                                 // +0.0f, ascending position
    for (int kb = 0; kb < cnt; kb += 16) {
      const int src = kb == 0 ? pos0 : (kb + hl < cnt ? __ldg(&c.perm[j0 + kb + hl]) : 0);
      const int m = min(16, cnt - kb);
      for (int k = 0; k < m; k += 4) {
        int p[4];
        float4 ga[4], gb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q] = __shfl_sync(hm, src, (k + q) & 15, 16);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ga[q] = zero; gb[q] = zero;
          if (k + q < m) {
            if (aa) ga[q] = __ldcs(G4 + (int64_t)p[q] * D4 + da);
            if (ab) gb[q] = __ldcs(G4 + (int64_t)p[q] * D4 + db);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (k + q < m) { acc0 = f4add_s(acc0, ga[q]); acc1 = f4add_s(acc1, gb[q]); }
      }
    }
    if (aa) {
      const float4 dl = f4scale_s(nlr, acc0);
      vr[da] = f4add_s(va, dl);
      pr[da] = f4add_s(pa, dl);   // clean: fl(+0 + delta) (R13)
    }
    if (ab) {
      const float4 dl = f4scale_s(nlr, acc1);
      vr[db] = f4add_s(vb, dl);
      pr[db] = f4add_s(pb, dl);
    }
  }
  if (hl == 0) s.cc[e] = ecc + 1;   // Cache.Clock
}

// ------------------------------------------------------------------ heavy rows -> hbuf
// Warp per 32 positions j: flag the heavy ones (cnt(inverse[perm[j]]) >
// SR_HEAVY), then copy their rows 8 at a time, one float4 per lane per row,
// into the slice-major buffer: hbuf[slice][j][16] = G[perm[j]][16 slice ...],
// so every (key, slice) item is one contiguous block of cnt x 64 B.
__global__ void __launch_bounds__(256) k_heavy_gather(Dev s, Call c, const float* __restrict__ G, int n) {
  Ctl* ctl = s.ctl;
  if (ctl->abort) return;
  const int lane = threadIdx.x & 31;
  const int D4 = s.D >> 2;
  const float4* G4 = reinterpret_cast<const float4*>(G);
  float4* H4 = reinterpret_cast<float4*>(c.hbuf);
  const int stride = gridDim.x * blockDim.x;
  for (int base = blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < n; base += stride) {
    const int j = base + lane;
    int p = 0;
    bool hv = false;
    if (j < n) {
      p = c.perm[j];
      const int u = c.inverse[p];
      hv = c.seg_off[u + 1] - c.seg_off[u] > SR_HEAVY;
    }
    unsigned m = __ballot_sync(0xffffffffu, hv);
    while (m) {
      int r[8], src[8], k = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        r[q] = m ? __ffs(m) - 1 : -1;
        if (m) { m &= m - 1; ++k; }
        src[q] = __shfl_sync(0xffffffffu, p, r[q] < 0 ? 0 : r[q]);
      }
      for (int d = lane; d < D4; d += 32) {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < k) v[q] = __ldcs(G4 + (int64_t)src[q] * D4 + d);
        // slice-major: float4 d of row j -> plane d / 4, row j, float4 d % 4
        float4* dst = H4 + (int64_t)(d >> 2) * c.hcap * 4 + (d & 3);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (q < k) __stcg(dst + (int64_t)(base + r[q]) * 4, v[q]);
      }
    }
  }
}

// Stage i of this CTA's stream: item = first item whose cumulative stage count
// exceeds i (items of the current batch of 32, one per lane).
struct StageRef {
  int item, u, j0, cnt, kb;
};
__device__ __forceinline__ StageRef stage_ref(int i, int scan, int u, int j0, int cnt, int SR) {
  StageRef r;
  r.item = __popc(__ballot_sync(0xffffffffu, scan <= i));
  const int before = r.item ? __shfl_sync(0xffffffffu, scan, (r.item - 1) & 31) : 0;
  r.u = __shfl_sync(0xffffffffu, u, r.item & 31);
  r.j0 = __shfl_sync(0xffffffffu, j0, r.item & 31);
  r.cnt = __shfl_sync(0xffffffffu, cnt, r.item & 31);
  r.kb = (i - before) * SR;
  return r;
}

// ---- optional instrumentation (-DHET_TIMELINE): per CTA [start, producer done,
// consumers done, stages, then (issue, ready) %globaltimer pairs of the first 120 stages]
#ifdef HET_TIMELINE
constexpr int SRT_W = 256;
__device__ unsigned long long g_srt[HV_CTAS * SRT_W];
__device__ __forceinline__ unsigned long long srt_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SRT(slot) g_srt[blockIdx.x * SRT_W + (slot)] = srt_now()
extern "C" int het_debug_timeline_sr(unsigned long long* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_srt, sizeof(g_srt));
  return HV_CTAS * SRT_W;
}
#else
#define SRT(slot) do {} while (0)
#endif

// Work items are (heavy key, 16-column slice), ordered by size bucket, largest
// first: item i = h * nsl + slice, h the key's rank in that order.  Items are
// dealt to the P pipelines in snake order (round r: pipeline gp takes item
// r * P + gp for even r, r * P + P - 1 - gp for odd r), which balances rows
// per pipeline to within one item of a power-of-two size class.  For one batch
// of 32 rounds (one item per lane): key, list entry, occurrence range, and the
// inclusive prefix of the items' stage counts.  bsz[b] = keys in bucket b.
struct Batch {
  int u, ent, j0, cnt, scan, total;
};
__device__ __forceinline__ Batch load_batch(const Call& c, const int* bsz, int round0, int gp, int P, int nitems,
                                            int cap, int nsl, int lane) {
  Batch b{0, 0, 0, 0, 0, 0};
  const int r = round0 + lane;
  const int item = r * P + ((r & 1) ? P - 1 - gp : gp);
  int nst = 0;
  if (item < nitems) {
    int h = item / nsl, bk = 31;
    while (h >= bsz[bk]) { h -= bsz[bk]; --bk; }
    b.ent = c.hlist[bucket_off(bk, cap) + h];
    b.u = b.ent & 0x7FFFFFFF;
    b.j0 = c.seg_off[b.u];
    b.cnt = c.seg_off[b.u + 1] - b.j0;
    nst = (b.cnt + HV_BR - 1) / HV_BR;
  }
  b.scan = nst;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, b.scan, o);
    if (lane >= o) b.scan += v;
  }
  b.total = __shfl_sync(0xffffffffu, b.scan, 31);
  return b;
}

__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_relaxed(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The producer path carries no release operation (fence / release arrive):
// on sm_100a those compile to MEMBAR.ALL.CTA, which waits for the thread's
// outstanding copies -- one stage in flight instead of four (measured).  The
// producer arrives relaxed; the consumer derives each stage's key, size and
// first/last flags from the same item list.
__global__ void __launch_bounds__(64 * HV_PIPES)
k_sr_heavy(Dev s, Call c, int cap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[HV_PIPES][HV_STAGES], empty[HV_PIPES][HV_STAGES];
  Ctl* ctl = s.ctl;
  if (ctl->abort) return;
  const int D = (int)s.D;
  const int nsl = (D + HV_W - 1) / HV_W;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int pipe = warp >> 1;                  // warps (2p, 2p+1) = (producer, consumer) of pipeline p
  const bool producer = (warp & 1) == 0;
  __shared__ int bsz[32];
  if (tid < 32) bsz[tid] = tid >= 5 ? ctl->nbucket[tid] : 0x7FFFFFFF;
  __syncthreads();
  int nh = 0;
  for (int q = 5; q < 32; ++q) nh += bsz[q];
  const int nitems = nh * nsl;
  const int P = HV_PIPES * (int)gridDim.x;
  const int gp = pipe * (int)gridDim.x + (int)blockIdx.x;
  float* ring = reinterpret_cast<float*>(smem) + (size_t)pipe * HV_STAGES * HV_BR * HV_W;   // [stage][row][16]
  if (tid == 0) {
    for (int q = 0; q < HV_PIPES; ++q)
      for (int i = 0; i < HV_STAGES; ++i) { mbar_init(&full[q][i], 1); mbar_init(&empty[q][i], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) SRT(0);
  uint32_t it = 0;   // stages of this pipeline
  const int nrounds = (nitems + P - 1) / P;
  for (int r0 = 0; r0 < nrounds; r0 += 32) {
    const Batch b = load_batch(c, bsz, r0, gp, P, nitems, cap, nsl, lane);
    float a = 0.f;
    for (int i = 0; i < b.total; ++i) {
      const StageRef r = stage_ref(i, b.scan, b.u, b.j0, b.cnt, HV_BR);
      const int rd = r0 + r.item;
      const int item = rd * P + ((rd & 1) ? P - 1 - gp : gp);
      const int col0 = (item % nsl) * HV_W;
      const uint32_t sl = it % HV_STAGES, k = it / HV_STAGES;
      float* stg = ring + (size_t)sl * HV_BR * HV_W;
      if (producer) {
        if (lane == 0) {
          if (k > 0) mbar_wait(&empty[pipe][sl], (k - 1) & 1);
          if (it < 120 && pipe == 0) SRT(4 + 2 * it);
          const int m = min(HV_BR, r.cnt - r.kb);
          mbar_expect_tx_relaxed(&full[pipe][sl], (uint32_t)m * HV_W * 4);
          mbar_arrive_relaxed(&full[pipe][sl]);
          bulk_g2s(stg, c.hbuf + ((int64_t)(col0 / HV_W) * c.hcap + r.j0 + r.kb) * HV_W, (uint32_t)m * HV_W * 4,
                   &full[pipe][sl]);
        }
      } else {
        const int m = min(HV_BR, r.cnt - r.kb);
        if (r.kb == 0) a = 0.f;                      // +0.0f, ascending position
        mbar_wait(&full[pipe][sl], k & 1);
        if (tid == 32 && it < 120) SRT(5 + 2 * it);
#ifdef HET_TIMELINE
        const long long lc0 = clock64();
#endif
        if (lane < HV_W) {
          // 16 rows in flight in registers: the next 16 load while these add
          const float* sp = stg + lane;
          int rr = 0;
          if (m >= 16) {
            float x[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) x[q] = sp[q * HV_W];
            for (rr = 16; rr + 16 <= m; rr += 16) {
              float y[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) y[q] = sp[(rr + q) * HV_W];
#pragma unroll
              for (int q = 0; q < 16; ++q) a = __fadd_rn(a, x[q]);
#pragma unroll
              for (int q = 0; q < 16; ++q) x[q] = y[q];
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) a = __fadd_rn(a, x[q]);
          }
          for (; rr < m; ++rr) a = __fadd_rn(a, sp[rr * HV_W]);
        }
        __syncwarp();
#ifdef HET_TIMELINE
        if (tid == 32 && it < 12) g_srt[blockIdx.x * SRT_W + 244 + it] = clock64() - lc0;
#endif
        if (lane == 0) mbar_arrive(&empty[pipe][sl]);
        // last stage: the slice's sums replace the item's first hbuf row
        // (already consumed); k_heavy_apply applies them
        if (r.kb + HV_BR >= r.cnt && lane < HV_W)
          c.hbuf[((int64_t)(col0 / HV_W) * c.hcap + r.j0) * HV_W + lane] = a;
      }
      ++it;
    }
  }
  if (tid == 0) {
    SRT(1);
#ifdef HET_TIMELINE
    g_srt[blockIdx.x * SRT_W + 3] = it;
#endif
  }
  if (tid == 32) SRT(2);
}

// ------------------------------------------------------------------ heavy keys: SGD + pending
// Thread per (heavy key, column): delta = (-lr) * acc, v += delta, p = (dirty ?
// p : +0) + delta (R13); acc sits in the key's first hbuf row of each slice.
__global__ void __launch_bounds__(256) k_heavy_apply(Dev s, Call c, float lr, int cap) {
  Ctl* ctl = s.ctl;
  if (ctl->abort) return;
  const int D = (int)s.D;
  const float nlr = -lr;
  for (int b = 5; b < 32; ++b) {
    const int nb = ctl->nbucket[b];
    const int off = bucket_off(b, cap);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nb * D;
         t += (int64_t)gridDim.x * blockDim.x) {
      const int h = (int)(t / D), d = (int)(t - (int64_t)h * D);
      const int32_t ent = c.hlist[off + h];
      const int u = ent & 0x7FFFFFFF;
      const int32_t e = c.uentry[u];
      const float acc = c.hbuf[((int64_t)(d / HV_W) * c.hcap + c.seg_off[u]) * HV_W + (d % HV_W)];
      const float dl = __fmul_rn(nlr, acc);
      const int64_t i = (int64_t)e * D + d;
      s.v[i] = __fadd_rn(s.v[i], dl);
      s.p[i] = __fadd_rn(ent < 0 ? s.p[i] : 0.f, dl);   // clean: fl(+0 + delta) (R13)
    }
  }
}

// ------------------------------------------------------------------ launcher
int launch_segreduce_apply(const Dev& s, const Call& c, const float* grads, float lr, int n, cudaStream_t st,
                           cudaStream_t side, cudaEvent_t fork, cudaEvent_t join) {
  static const bool no_heavy = getenv("HET_SR_NO_HEAVY") != nullptr;   // diagnostic: light kernel only
  const bool heavy_path = !no_heavy && n > SR_HEAVY && side && fork && join;
  int launches = 0;
  if (heavy_path) {
    const size_t smem = (size_t)HV_PIPES * HV_STAGES * HV_BR * HV_W * 4;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_sr_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    cudaMemsetAsync(s.ctl->nbucket, 0, sizeof(s.ctl->nbucket), st);
    const int lb = std::min(148 * 4, std::max(1, (n + 255) / 256));
    k_heavy_list<<<lb, 256, 0, st>>>(s, c, n);
    cudaEventRecord(fork, st);
    cudaStreamWaitEvent(side, fork, 0);
    k_heavy_gather<<<std::min(148 * 8, std::max(1, (n + 255) / 256)), 256, 0, side>>>(s, c, grads, n);
    k_sr_heavy<<<HV_CTAS, 64 * HV_PIPES, smem, side>>>(s, c, n);
    k_heavy_apply<<<148 * 2, 256, 0, side>>>(s, c, lr, n);
    cudaEventRecord(join, side);
    launches += 4;
  }
  const int blocks = std::max(1, (n + LT_THREADS / 16 - 1) / (LT_THREADS / 16));
  k_sr_light<<<blocks, LT_THREADS, 0, st>>>(s, c, grads, lr, heavy_path ? SR_HEAVY : INT_MAX);
  launches += 1;
  if (heavy_path) cudaStreamWaitEvent(st, join, 0);
  return launches;
}

}  // namespace het
