// Dependent random-load latency over arrays of growing size (TLB / DRAM reach).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe latency_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void chase(const uint64_t* __restrict__ next, uint64_t start, int steps, uint64_t* out, long long* cyc) {
  uint64_t p = start;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = next[p];
  long long t1 = clock64();
  *out = p;
  *cyc = t1 - t0;
}

__global__ void init(uint64_t* a, uint64_t n, uint64_t stride_elems, uint64_t seed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    a[i] = (x % (n / stride_elems)) * stride_elems;   // random element on another 4 KB-strided slot
  }
}

int main() {
  const size_t sizes_mb[] = {16, 64, 256, 1024, 4096, 16384};
  uint64_t* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  for (size_t mb : sizes_mb) {
    size_t n = mb * (1ull << 20) / 8;
    uint64_t* a;
    if (cudaMalloc(&a, n * 8) != cudaSuccess) { printf("alloc %zu MB failed\n", mb); break; }
    init<<<1024, 256>>>(a, n, 512, 12345);   // 4 KB strided targets
    cudaDeviceSynchronize();
    chase<<<1, 1>>>(a, 0, 200, out, cyc);      // warm
    chase<<<1, 1>>>(a, 7 * 512, 4000, out, cyc);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("array %6zu MB: %.0f cycles per dependent load\n", mb, (double)c / 4000);
    cudaFree(a);
  }
  return 0;
}
