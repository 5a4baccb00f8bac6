// tcgen05.ld throughput: 4 warps (one per lane quadrant) each loading 32x32b.x32 repeatedly.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(float* out, long long* cyc, int iters, int nwarps_active) {
  __shared__ uint32_t slot;
  int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float acc = 0;
  long long t0 = clock64();
  if (warp < nwarps_active) {
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
        : "r"(base + (it & 7) * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(slot));
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 64);
  for (int nw : {1, 4, 8}) {
    int iters = 1000; long long h;
    k<<<1, 256>>>(out, cyc, iters, nw); cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double bytes = (double)iters * 4096 * nw;
    printf("%d warps: %lld cyc, %.1f B/clk/SM (x32 ld + wait each) %s\n", nw, h, bytes / h, cudaGetErrorString(e));
  }
  return 0;
}
