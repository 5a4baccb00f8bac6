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

// The barrier protocol, executed by one warp for rank `rank`: fence this rank's prior stores
// system-wide, bump the local epoch, release-store it into every rank's flag word for this
// rank, then acquire-spin until every rank's word for us reaches the epoch (trap on timeout).
__device__ __forceinline__ void barrier_warp(uint32_t* const* flags, uint32_t* epoch, int rank, int world,
                                             unsigned long long timeout_ns) {
  __threadfence_system();
  __syncwarp();
  uint32_t e = 0;
  if (threadIdx.x % 32 == 0) {
    e = *epoch + 1;
    *epoch = e;
  }
  e = __shfl_sync(0xffffffffu, e, 0);
  const int i = threadIdx.x % 32;
  if (i < world) {
    uint32_t* dst = flags[i] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(dst), "r"(e) : "memory");
    const uint32_t* mine = flags[rank] + i;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if ((int)(v - e) >= 0) break;
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > timeout_ns) {
        printf("ftb_peer_barrier: rank %d timed out waiting for rank %d (epoch %u, saw %u)\n", rank, i, e, v);
        __trap();
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
}

__global__ void peer_barrier_kernel(const BarrierParams p) {
  barrier_warp(p.flags, p.epoch, p.rank, p.world, p.timeout_ns);
}

// Self-test of the protocol with truly concurrent ranks on ONE device: block b plays rank b
// (cooperative launch: all blocks co-resident, so the ranks' spins cannot starve one another).
// Per round every rank writes a payload word, passes the barrier, and checks every rank's
// payload of that round (it must be visible after the barrier); mismatches are counted.
struct SelftestParams {
  uint32_t* flags[FTB_MAX_PEERS];
  uint32_t* epochs;   // [world]
  uint32_t* data;     // [rounds][world]
  uint32_t* errors;   // [1]
  int world, rounds;
  unsigned long long timeout_ns;
};

__global__ void peer_barrier_selftest_kernel(const SelftestParams p) {
  const int rank = blockIdx.x;
  for (int r = 0; r < p.rounds; ++r) {
    if (threadIdx.x == 0) p.data[(size_t)r * p.world + rank] = (uint32_t)(r * 131 + rank * 7 + 1);
    barrier_warp(p.flags, p.epochs + rank, rank, p.world, p.timeout_ns);
    const int i = threadIdx.x;
    if (i < p.world) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p.data + (size_t)r * p.world + i) : "memory");
      if (v != (uint32_t)(r * 131 + i * 7 + 1)) atomicAdd(p.errors, 1u);
    }
    // second barrier: nobody overwrites round r+1's slot reuse before all checked round r
    barrier_warp(p.flags, p.epochs + rank, rank, p.world, p.timeout_ns);
  }
}

extern "C" int ftb_peer_barrier_selftest(int32_t world, int32_t rounds, uint32_t* flags, uint32_t* epochs,
                                         uint32_t* data, uint32_t* errors, double timeout_s, void* stream) {
  if (world < 1 || world > FTB_MAX_PEERS || rounds < 1 || !flags || !epochs || !data || !errors)
    return set_error(FTB_EINVAL, "peer_barrier_selftest: bad arguments");
  SelftestParams p{};
  for (int i = 0; i < world; ++i) p.flags[i] = flags + (size_t)i * world;
  p.epochs = epochs;
  p.data = data;
  p.errors = errors;
  p.world = world;
  p.rounds = rounds;
  p.timeout_ns = (unsigned long long)((timeout_s > 0 ? timeout_s : 10.0) * 1e9);
  void* args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)peer_barrier_selftest_kernel, dim3(world), dim3(32), args, 0,
                                              reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_cuda_error(e, "peer_barrier_selftest launch");
  return check_launch("peer_barrier_selftest_kernel");
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
