// Issue throughput (lanes/clk/SM) of the softmax inner-loop instructions on B200:
// MUFU.EX2, F2FP bf16x2 pack, integer round+PRMT pack, FMNMX3, FFMA2, FADD2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/pipes.cu -o scripts/micro/pipes_bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint32_t prmt2(float a, float b) {
  uint32_t r;
  asm volatile("{ .reg .u32 x, y; add.u32 x, %1, 0x8000; add.u32 y, %2, 0x8000; prmt.b32 %0, x, y, 0x7632; }"
               : "=r"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
  return r;
}
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float max3(float a, float b, float c) { float d; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
  float a[16];
  uint32_t u = 0;
  for (int i = 0; i < 16; ++i) a[i] = 0.01f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) { a[i] = ex2(a[i]); a[i + 1] = ex2(a[i + 1]); }
      if (MODE == 1) { u ^= cvt2(a[i], a[i + 1]); a[i] += 1e-7f; }
      if (MODE == 2) { u ^= prmt2(a[i], a[i + 1]); a[i] += 1e-7f; }
      if (MODE == 3) { a[i] = max3(a[i], a[i + 1], a[(i + 2) & 15]); }
      if (MODE == 4) { uint32_t t = ex2h2(__float_as_uint(a[i])); a[i] = __uint_as_float(t ^ 0x3c00u); }
      if (MODE == 5) { uint32_t t = ex2bf2(__float_as_uint(a[i])); a[i] = __uint_as_float(t ^ 0x3f80u); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = __uint_as_float(u); for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const char* names[6] = {"MUFU.EX2 (per elem)", "F2FP pack + FADD (per pair)", "IADD x2 + PRMT pack + FADD (per pair)",
                          "FMNMX3 (per instr)", "ex2.approx.f16x2 (per instr = 2 elem)", "ex2.approx.ftz.bf16x2 (per instr)"};
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int m = 0; m < 6; ++m) {
      long long h;
      if (m == 0) k<0><<<1, 32 * warps>>>(out, cyc, 1000);
      if (m == 1) k<1><<<1, 32 * warps>>>(out, cyc, 1000);
      if (m == 2) k<2><<<1, 32 * warps>>>(out, cyc, 1000);
      if (m == 3) k<3><<<1, 32 * warps>>>(out, cyc, 1000);
      if (m == 4) k<4><<<1, 32 * warps>>>(out, cyc, 1000);
      if (m == 5) k<5><<<1, 32 * warps>>>(out, cyc, 1000);
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      double n = 1000.0 * (m == 0 ? 16 : 8) * 32 * warps;
      printf("warps %2d  %-40s %.2f ops/clk/SM\n", warps, names[m], n / h);
    }
  }
  return 0;
}
