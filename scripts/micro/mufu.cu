// MUFU.EX2 vs FFMA2-polynomial throughput on one SM (clock64), B200 measurement.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.01f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.5f;
      else a[i] = fmaf(fmaf(fmaf(a[i], 0.05f, 0.24f), a[i], 0.69f), a[i], 1.0f) - 1.5f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  for (int warps = 1; warps <= 16; warps *= 2) {
    long long h[2];
    k<0><<<1, 32 * warps>>>(out, cyc, 1000); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    k<1><<<1, 32 * warps>>>(out, cyc, 1000); cudaMemcpy(h + 1, cyc, 8, cudaMemcpyDeviceToHost);
    double n = 1000.0 * 16 * 32 * warps;
    printf("warps %2d: ex2 %.2f lanes/clk/SM   poly(3 FMA) %.2f lanes/clk/SM\n", warps, n / h[0], n / h[1]);
  }
  return 0;
}
