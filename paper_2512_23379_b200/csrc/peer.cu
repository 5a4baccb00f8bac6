// Peer memory for the fused Ulysses exchange: IPC-exportable device
// allocations, their import on the other ranks of the node (NVLink / NVSwitch
// peer mappings), and a stream-ordered cross-rank barrier kernel.
//
// The producer kernels (QKV GEMM epilogue, FMHA epilogue, out-projection epilogue)
// store straight into the peers' receive buffers; one barrier after each producer
// makes the stores visible before any consumer reads. Two barriers per layer also
// guard buffer reuse across layers (a rank cannot start layer l+1's stores until
// every rank has passed layer l's consumer).
#include <stdio.h>

#include "ftb_internal.h"

using namespace ftb;

static_assert(sizeof(cudaIpcMemHandle_t) == FTB_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" int ftb_sym_alloc(size_t bytes, void** ptr) {
  if (!ptr || !bytes) return set_error(FTB_EINVAL, "sym_alloc: bad arguments");
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, "sym_alloc");
  e = cudaMemset(*ptr, 0, bytes);
  if (e != cudaSuccess) return set_cuda_error(e, "sym_alloc memset");
  return FTB_OK;
}

extern "C" int ftb_sym_free(void* ptr) {
  if (!ptr) return FTB_OK;
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? FTB_OK : set_cuda_error(e, "sym_free");
}

extern "C" int ftb_ipc_export(const void* ptr, uint8_t* handle) {
  if (!ptr || !handle) return set_error(FTB_EINVAL, "ipc_export: bad arguments");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(ptr));
  if (e != cudaSuccess) return set_cuda_error(e, "ipc_export");
  memcpy(handle, &h, sizeof(h));
  return FTB_OK;
}

extern "C" int ftb_ipc_import(const uint8_t* handle, void** ptr) {
  if (!ptr || !handle) return set_error(FTB_EINVAL, "ipc_import: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_cuda_error(e, "ipc_import");
  return FTB_OK;
}

extern "C" int ftb_ipc_close(void* ptr) {
  if (!ptr) return FTB_OK;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? FTB_OK : set_cuda_error(e, "ipc_close");
}

extern "C" int ftb_copy_d2d(void* dst, const void* src, size_t bytes, void* stream) {
  if (!dst || !src) return set_error(FTB_EINVAL, "copy_d2d: null pointer");
  if (!bytes) return FTB_OK;
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FTB_OK : set_cuda_error(e, "copy_d2d");
}

extern "C" int ftb_copy_d2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                               void* stream) {
  if (!dst || !src || width > dpitch || width > spitch) return set_error(FTB_EINVAL, "copy_d2d_2d: bad arguments");
  if (!width || !height) return FTB_OK;
  cudaError_t e = cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice,
                                    reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FTB_OK : set_cuda_error(e, "copy_d2d_2d");
}

struct BarrierParams {
  uint32_t* flags[FTB_MAX_PEERS];  // rank i's flag words [world]; flags[i][r] = last epoch rank r signalled i
  uint32_t* epoch;                 // this rank's local epoch counter (device word)
  int rank, world;
  unsigned long long timeout_ns;
};

__global__ void peer_barrier_kernel(const BarrierParams p) {
  __shared__ uint32_t e_sh;
  // make every store this rank issued before the barrier (previous kernels on the
  // stream, peer-mapped or local) visible system-wide before signalling
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t e = *p.epoch + 1;
    *p.epoch = e;
    e_sh = e;
  }
  __syncthreads();
  const uint32_t e = e_sh;
  const int i = threadIdx.x;
  if (i < p.world) {
    uint32_t* dst = p.flags[i] + p.rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(e) : "memory");
    const uint32_t* mine = p.flags[p.rank] + i;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int)(v - e) >= 0) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > p.timeout_ns) {
        printf("ftb_peer_barrier: rank %d timed out waiting for rank %d (epoch %u, saw %u)\n", p.rank, i, e, v);
        __trap();
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

extern "C" int ftb_peer_barrier(uint32_t* const* flags, uint32_t* epoch, int32_t rank, int32_t world,
                                double timeout_s, void* stream) {
  if (!flags || !epoch || world < 1 || world > FTB_MAX_PEERS || rank < 0 || rank >= world)
    return set_error(FTB_EINVAL, "peer_barrier: bad arguments");
  BarrierParams p{};
  for (int i = 0; i < world; ++i) {
    if (!flags[i]) return set_error(FTB_EINVAL, "peer_barrier: null flag pointer");
    p.flags[i] = flags[i];
  }
  p.epoch = epoch;
  p.rank = rank;
  p.world = world;
  p.timeout_ns = (unsigned long long)((timeout_s > 0 ? timeout_s : 30.0) * 1e9);
  peer_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  return check_launch("peer_barrier_kernel");
}
