// Internal host-side helpers shared by the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/ftb2.h"

namespace ftb {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_launch(const char* what);
int sm_count();
// bf16 tensor map, SWIZZLE_128B, OOB -> zero. dims/box innermost first; strides in bytes (rank-1 entries).
int make_tmap_bf16(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                   const uint32_t* box, int swizzle_bytes = 128);
// fp32 2-D/3-D tensor map (same conventions as make_tmap_bf16; swizzle 128 B).
int make_tmap_f32(CUtensorMap* map, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
                  const uint32_t* box);
}  // namespace ftb
