// Ordered column-sum loop from k_sr_heavy's consumer, in isolation: one warp,
// 16 (or 32) active lanes, 256 rows of a [row][W] shared-memory tile, repeated.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_bench chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int MODE>
__global__ void chain(float* out, long long* cyc, int reps, int mrt) {
  __shared__ float stg[256 * 32];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) stg[i] = 1e-3f * (i % 97);
  __syncthreads();
  float a = 0.f;
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (lane < W) {
      const float* sp = stg + lane;
      const int m = MODE >= 10 ? mrt : 256;
      if (MODE == 0) {   // simple
#pragma unroll 8
        for (int rr = 0; rr < m; ++rr) a = __fadd_rn(a, sp[rr * W]);
      } else if (MODE == 1 || MODE == 11) {   // 16-deep register pipeline (kernel's loop)
        int rr = 0;
        float x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = sp[q * W];
        for (rr = 16; rr + 16 <= m; rr += 16) {
          float y[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) y[q] = sp[(rr + q) * W];
#pragma unroll
          for (int q = 0; q < 16; ++q) a = __fadd_rn(a, x[q]);
#pragma unroll
          for (int q = 0; q < 16; ++q) x[q] = y[q];
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) a = __fadd_rn(a, x[q]);
      } else {   // plain +, fully unrolled by 32
#pragma unroll 32
        for (int rr = 0; rr < m; ++rr) a += sp[rr * W];
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int W, int MODE>
void run(const char* name, float* out, long long* cyc) {
  const int reps = 200;
  chain<W, MODE><<<1, 32>>>(out, cyc, reps, 256);
  chain<W, MODE><<<1, 32>>>(out, cyc, reps, 256);
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.2f cycles/row\n", name, (double)c / (reps * 256.0));
}

int main() {
  float* out; long long* cyc;
  cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
  run<16, 0>("W16 simple unroll8", out, cyc);
  run<16, 1>("W16 16-deep pipeline", out, cyc);
  run<16, 2>("W16 plain + unroll32", out, cyc);
  run<32, 1>("W32 16-deep pipeline", out, cyc);
  run<16, 11>("W16 16-deep runtime m", out, cyc);
  return 0;
}
