// tcgen05.mma cta_group::2 throughput per SM pair: M=256 (128 rows per SM), K=16 bf16,
// N in {128, 256}, A from smem (SS) or TMEM (TS). One cluster of 2 CTAs per SM pair, the
// leader's thread 0 issues. Compare with scripts/micro/mma.cu (1-CTA, M=128).
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I paper_2512_23379_b200/csrc scripts/micro/mma_pair.cu
#include <cstdio>
#include "common.cuh"
using namespace ftb;

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(long long* cyc, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 16384);
    constexpr uint32_t id = idesc_bf16(256, N, 0, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t off = (i & 3) * 32;
      if (TS)
        asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(tmem),
                     "r"(tmem + 256 + (i & 7) * 8), "l"(sdesc_sw128(sb + off, 16, 1024)), "r"(id));
      else
        mma_bf16_ss_pair(tmem, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), id, 1u);
    }
    mma_commit_pair(&bar, 0x3);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    cyc[blockIdx.x >> 1] = t1 - t0;
  }
  if (threadIdx.x == 0 && rank == 1) mbar_wait(&bar, 0);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 0) tmem_dealloc_pair<512>(tmem);
}

template <int N, bool TS>
void run(long long* cyc) {
  const int iters = 4096;
  cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<N, TS><<<148, 128, 65536>>>(cyc, iters);
  k<N, TS><<<148, 128, 65536>>>(cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[74];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 74; ++i) avg += h[i];
  avg /= 74;
  const double flops = 2.0 * 128 * N * 16;  // per SM
  printf("pair %s M=256 N=%3d K=16: %.1f clk/mma, %.0f flop/clk/SM (%s)\n", TS ? "TS" : "SS", N, avg / iters,
         flops * iters / avg, cudaGetErrorString(e));
}

int main() {
  long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<128, false>(cyc);
  run<256, false>(cyc);
  run<128, true>(cyc);
  run<256, true>(cyc);
  return 0;
}
