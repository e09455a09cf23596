// Row-gather ring microbenchmark: each CTA streams `rows` rows of 512 B chosen
// by an index list (stride-26 pattern, like one Criteo field's occurrences)
// through an 8-stage shared-memory ring; 4 consumer warps sum columns.
// Producer variants: 0 = cp.async (LDGSTS) 2 warps, 1 = cp.async 4 warps,
// 2 = cp.async.bulk per row (no fence), 3 = LDG.128 -> STS by 4 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ring_bench ring_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

constexpr int NS = 8, SR = 32, D = 128, CONS = 4;

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t done;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
  } while (!done);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* b) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_relaxed(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}

template <int V, int PROD, bool SUM, int SRX = SR>
__global__ void ring(const float* __restrict__ G, const int* __restrict__ idx, int rows, float* out, size_t n_rows) {
  extern __shared__ __align__(128) float stg[];
  __shared__ uint64_t full[NS], empty[NS];
  int* sidx = reinterpret_cast<int*>(stg + (size_t)NS * SR * D);   // all indices, preloaded
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int* my = idx + (size_t)blockIdx.x * rows;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], (V == 2 || V == 6 || V == 7) ? 1 : (V == 3 ? PROD * 32 : 32 * PROD));
      mbar_init(&empty[i], CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < rows; i += blockDim.x) sidx[i] = my[i];
  __syncthreads();
  const int nst = rows / SR;
  if (warp < PROD && (V == 4 || V == 5)) {
    constexpr int W = V == 4 ? 128 : 32;        // floats per row slice
    constexpr int W4 = W / 4;
    constexpr int RPL = SRX / 32;               // rows per lane per stage
    const int nstx = rows / SRX;
    int curx[8][RPL], nxtx[8][RPL];
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int j = 0; j < RPL; ++j) curx[q][j] = __ldg(&my[q * SRX + j * 32 + lane]);
    for (int g = 0; g < nstx; g += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < RPL; ++j) nxtx[q][j] = (g + 8 + q) < nstx ? __ldg(&my[(g + 8 + q) * SRX + j * 32 + lane]) : 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int it = g + q;
        const int sl = it % NS, k = it / NS;
        if (k > 0) mbar_wait(&empty[sl], (k - 1) & 1);
        float* dst = stg + (size_t)sl * SR * D;
#pragma unroll
        for (int ch0 = warp * 32; ch0 < SRX * W4; ch0 += 32 * PROD) {
          const int ch = ch0 + lane;
          const int row = ch / W4, q4 = ch % W4;
          int src = 0;
#pragma unroll
          for (int j = 0; j < RPL; ++j) { const int t = __shfl_sync(0xffffffffu, curx[q][j], row & 31); if ((row >> 5) == j) src = t; }
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst + row * W + 4 * q4)),
                       "l"(G + (size_t)src * D + 4 * q4) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[sl])) : "memory");
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int j = 0; j < RPL; ++j) curx[q][j] = nxtx[q][j];
    }
  } else if (warp < PROD) {
    for (int it = 0; it < nst; ++it) {
      const int sl = it % NS, k = it / NS;
      if (k > 0) mbar_wait(&empty[sl], (k - 1) & 1);
      float* dst = stg + (size_t)sl * SR * D;
      const int src_l = sidx[it * SR + lane];
      if (V == 4 || V == 5) {
        // handled below (register-prefetched indices)
      } else if (V == 6 || V == 7) {
        if (lane == 0) {
          mbar_expect_tx_relaxed(&full[sl], SR * D * 4);
          mbar_arrive_relaxed(&full[sl]);
          const size_t row0 = ((size_t)blockIdx.x * rows + (size_t)it * SR) % (n_rows - SR);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           sa(dst)), "l"(G + row0 * D + (V == 7 ? 16 : 0)), "r"(SR * D * 4), "r"(sa(&full[sl])) : "memory");
        }
      } else if (V == 0) {
        for (int r = warp; r < SR; r += PROD) {
          const int src = __shfl_sync(0xffffffffu, src_l, r);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(dst + r * D + 4 * lane)),
                       "l"(G + (size_t)src * D + 4 * lane) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(&full[sl])) : "memory");
      } else if (V == 2) {
        if (lane == 0) {
          mbar_expect_tx_relaxed(&full[sl], SR * D * 4);
          mbar_arrive_relaxed(&full[sl]);
        }
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(dst + lane * D)), "l"(G + (size_t)src_l * D), "r"(D * 4), "r"(sa(&full[sl])) : "memory");
      } else {
        float4 v[SR / PROD];
#pragma unroll
        for (int j = 0; j < SR / PROD; ++j) {
          const int src = __shfl_sync(0xffffffffu, src_l, warp + j * PROD);
          v[j] = __ldcs(reinterpret_cast<const float4*>(G + (size_t)src * D) + lane);
        }
#pragma unroll
        for (int j = 0; j < SR / PROD; ++j) reinterpret_cast<float4*>(dst + (warp + j * PROD) * D)[lane] = v[j];
        mbar_arrive(&full[sl]);   // every producer thread (release: its STS)
      }
    }
  } else {
    const int ct = tid - 32 * PROD;
    float a = 0.f;
    if (V == 5) {
      const int nstx = rows / SRX;
      for (int it = 0; it < nstx; ++it) {
        const int sl = it % NS, k = it / NS;
        mbar_wait(&full[sl], k & 1);
        const float* s = stg + (size_t)sl * SR * D;
        if (ct < 32) {
#pragma unroll 8
          for (int r = 0; r < SRX; ++r) a = __fadd_rn(a, s[r * 32 + ct]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sl]);
      }
      out[blockIdx.x * D + ct] = a;
      return;
    }
    for (int it = 0; it < nst; ++it) {
      const int sl = it % NS, k = it / NS;
      mbar_wait(&full[sl], k & 1);
      const float* s = stg + (size_t)sl * SR * D;
      if (SUM) {
#pragma unroll 8
        for (int r = 0; r < SR; ++r) a = __fadd_rn(a, s[r * D + ct]);
      } else {
        a += s[ct];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
    out[blockIdx.x * D + ct] = a;
  }
}

template <int V, int PROD, bool SUM, int SRX = SR>
float run(const float* G, const int* idx, int rows, int ctas, float* out) {
  const size_t smem = (size_t)NS * SR * D * 4 + (size_t)rows * 4;
  cudaFuncSetAttribute(ring<V, PROD, SUM, SRX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  ring<V, PROD, SUM, SRX><<<ctas, 32 * (PROD + CONS), smem>>>(G, idx, rows, out, 851968);
  cudaEventRecord(a);
  ring<V, PROD, SUM, SRX><<<ctas, 32 * (PROD + CONS), smem>>>(G, idx, rows, out, 851968);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) printf("err %s\n", cudaGetErrorString(e));
  return ms;
}

int main() {
  const size_t n = 851968;                      // rows of G (batch 32768 x 26 fields)
  float* G; cudaMalloc(&G, n * D * 4); cudaMemset(G, 0, n * D * 4);
  float* out; cudaMalloc(&out, 148 * D * 4);
  const int rows = 16384;   // 64 KB of indices + 128 KB ring
  for (int pat = 0; pat < 1; ++pat)
  for (int ctas : {1, 148}) {
    std::vector<int> h((size_t)ctas * rows);
    uint64_t x = 88172645463325252ull;
    for (int c = 0; c < ctas; ++c)
      for (int r = 0; r < rows; ++r) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        h[(size_t)c * rows + r] = pat == 0 ? (int)(((size_t)r * 26 + c % 26 + (size_t)c * 7919) % n)
                                           : (int)(x % n);                      // random rows
      }
    printf("pattern %s\n", pat == 0 ? "stride-26" : "random");
    int* idx; cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const double bytes = (double)ctas * rows * D * 4;   // (slice variants move 1/4 of this)
    auto rep = [&](const char* name, float ms) {
      printf("ctas %3d %-22s %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA\n", ctas, name, ms * 1e3,
             bytes / (ms * 1e-3) / 1e9, bytes / ctas / (ms * 1e-3) / 1e9);
    };
    const double q = 0.25;
    auto rep4 = [&](const char* name, float ms) {
      printf("ctas %3d %-26s %8.1f us  %7.1f GB/s total  %6.1f GB/s per CTA\n", ctas, name, ms * 1e3,
             q * bytes / (ms * 1e-3) / 1e9, q * bytes / ctas / (ms * 1e-3) / 1e9);
    };
    rep("bulk 16KB contiguous", run<6, 1, true>(G, idx, rows, ctas, out));
    rep("bulk 16KB contig +64B", run<7, 1, true>(G, idx, rows, ctas, out));
    cudaFree(idx);
  }
  return 0;
}
