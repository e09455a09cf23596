// Probe: DRAM -> shared-memory ingest rate of cp.async.bulk (one issuing
// thread per CTA, a ring of stages, nothing consumed) versus plain 128-bit
// loads, for random row-sized chunks of a multi-GB buffer, by chunk size,
// stages in flight and CTAs per SM.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t hsh(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}

__global__ void tma_read(const char* src, uint64_t nchunks, int chunk, int per_cta, int stages, int* sink) {
  extern __shared__ __align__(1024) char ring_all[];
  __shared__ __align__(8) uint64_t full_all[8][16];
  const int w = threadIdx.x >> 5;   // issuing warp: its own ring and barriers
  uint64_t* full = full_all[w];
  char* ring = ring_all + (size_t)w * stages * chunk;
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if ((threadIdx.x & 31) != 0) return;
  const uint64_t base = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + w) * per_cta;
  uint32_t ph[16] = {0};
  for (int i = 0; i < per_cta; ++i) {
    const int sl = i % stages;
    if (i >= stages) {   // wait for this slot's previous copy
      uint32_t done = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(su32(&full[sl])), "r"(ph[sl]) : "memory");
      } while (!done);
      ph[sl] ^= 1;
    }
    const uint64_t r = hsh(base + i) % nchunks;
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[sl])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(ring + (size_t)sl * chunk)), "l"(src + r * chunk), "r"(chunk), "r"(su32(&full[sl])) : "memory");
  }
  for (int i = 0; i < stages && i < per_cta; ++i) {
    const int sl = (per_cta - 1 - i) % stages;
    uint32_t done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(su32(&full[sl])), "r"(ph[sl]) : "memory");
    } while (!done);
    ph[sl] ^= 1;
  }
  if (ring[0] == 123) *sink = 1;
}

// plain loads: warp per chunk, 4 x 16 B per lane in flight
__global__ void ldg_read(const float4* src, uint64_t nchunks, int chunk, int per_warp, int* sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int c4 = chunk / 16;
  float acc = 0.f;
  for (int i = 0; i < per_warp; ++i) {
    const uint64_t r = hsh(w * per_warp + i) % nchunks;
    const float4* p = src + r * c4;
    for (int d = lane; d < c4; d += 128) {
      float4 a[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) a[b] = d + 32 * b < c4 ? __ldcs(p + d + 32 * b) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int b = 0; b < 4; ++b) acc += a[b].x;
    }
  }
  if (acc == 12345.f) *sink = 1;
}

int main() {
  const size_t bytes = 8ull << 30;
  char* src;
  int* sink;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  cudaMalloc(&sink, 4);
  char* fl;
  cudaMalloc(&fl, 256 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t total = 128ull << 20;   // bytes moved per measurement
  for (int chunk : {1024, 2048, 4096, 16384}) {
    for (int cps : {1, 2, 4}) {
      for (int W : {1, 2, 4, 8}) {
        const int stages = 4;
        const size_t smem = (size_t)W * stages * chunk;
        if (smem * cps > 220 * 1024) continue;
        const int ctas = sms * cps;
        const int per = (int)(total / chunk / ctas / W);
        cudaMemsetAsync(fl, 1, 256 << 20);
        cudaEventRecord(a);
        tma_read<<<ctas, 32 * W, smem>>>(src, bytes / chunk, chunk, per, stages, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("tma chunk %6d ctas/SM %d issuing warps/CTA %d stages %d: %7.1f GB/s\n", chunk, cps, W, stages,
               per * (double)chunk * ctas * W / ms / 1e6);
      }
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
