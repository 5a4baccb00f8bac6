// Causal 3D convolution as an implicit GEMM on tcgen05 (wan-mode VAE decoder).
//
//   out[t, y, x, n] = bias[n] + sum_{dt,dy,dx,c} in[t+dt+t0, y+dy-ph, x+dx-pw, c] * W[n, (dt,dy,dx), c]
//
// Activations are channel-last bf16 [T][H][W][C]; the causal time padding is
// the 2 cached frames the caller keeps in front of the current chunk's frames
// (t0 = 0 with a KT=3 kernel reads frames t, t+1, t+2 of the padded buffer).
// An M tile is 128 consecutive output pixels of one (t, y) row (tiles ordered x, t, y so
// consecutive tiles re-read the same input rows from L2); for every tap
// the producer issues one 4D TMA box {BK channels, 128 px, 1 row, 1 frame} at
// the shifted coordinates — spatial zero padding is the TMA out-of-bounds
// fill. The B operand is W^T [Cout][taps*Cin] (K-major). Same warp-specialised
// pipeline as gemm.cu (TMA warp, single-thread MMA issuer, 4 epilogue warps,
// double-buffered TMEM accumulators). Epilogue modes: bias (+ residual) bf16
// store; time-split store for the temporal x2 upsample conv; RGB8 for the head.
#include "common.cuh"
#include "ftb_internal.h"

namespace ftb {

struct ConvParams {
  int T, H, W, Cin, Cout;
  int KT, KH, KW, t0, pad_h, pad_w;
  int num_xt, kb_per_tap, taps;
  const float* bias;
  const __nv_bfloat16* resid;
  long long resid_ld;
  void* out;
  long long out_ld;
  int mode;       // 0 store, 1 time split, 2 RGB8
  int out_f32;    // mode bit 4: fp32 output
  int resid_f32;  // mode bit 5: fp32 residual
  int halo;       // dx-reuse kernel: rows -1 / H come from the halo maps (spatial split)
  // fused RMS norm (+SiLU) of the output pixel over all Cout channels (one N tile):
  // norm_out[pix*norm_ld + c] = bf16(silu(v_c * sqrt(Cout) / max(||v||, eps) * gamma_c))
  const float* norm_gamma;
  __nv_bfloat16* norm_out;
  long long norm_ld;
  int norm_silu;
  int write_main;  // 0: only the normalised output (the raw conv output has no other consumer)
};

template <int BN, int BK>
struct ConvCfg {
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196 * 1024) / STAGE_BYTES > 8 ? 8 : (196 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 64) ? 64 : ((2 * BN <= 128) ? 128 : ((2 * BN <= 256) ? 256 : 512));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t LAYOUT = (BK == 64) ? 2u : 4u;  // SW128 / SW64
  static constexpr uint32_t SBO = 8 * BK * 2;               // 8 rows of one swizzle atom
};

// acc -> + bias (+ residual) for the norm path (mode 0, full 32-column chunks)
__device__ __forceinline__ void conv_epilogue_values(const ConvParams& p, int t, int y, int x, int gc0,
                                                     float (&v)[32]) {
  if (p.bias) {  // float4 loads: 32 scalar broadcast loads each stalled their FADD (ncu)
    const float4* b4 = reinterpret_cast<const float4*>(p.bias + gc0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = __ldg(b4 + q);
      v[4 * q] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
  }
  if (p.resid) {
    const long long pix = ((long long)t * p.H + y) * p.W + x;
    if (p.resid_f32) {
      const float4* r = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.resid) + pix * p.resid_ld + gc0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 f = r[q];
        v[4 * q] += f.x;
        v[4 * q + 1] += f.y;
        v[4 * q + 2] += f.z;
        v[4 * q + 3] += f.w;
      }
    } else {
      const __nv_bfloat16* r = p.resid + pix * p.resid_ld + gc0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 w = *reinterpret_cast<const uint4*>(r + 8 * q);
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h2[e]);
          v[8 * q + 2 * e] += f.x;
          v[8 * q + 2 * e + 1] += f.y;
        }
      }
    }
  }
}

// main store of a finished chunk (mode 0)
__device__ __forceinline__ void conv_store(const ConvParams& p, int t, int y, int x, int gc0, const float (&v)[32]) {
  const long long pix = ((long long)t * p.H + y) * p.W + x;
  if (p.out_f32) {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + pix * p.out_ld + gc0);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return;
  }
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + pix * p.out_ld + gc0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 w;
    w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
    w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
    w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
    w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
    reinterpret_cast<uint4*>(o)[q] = w;
  }
}

__device__ __forceinline__ void conv_epilogue(const ConvParams& p, int t, int y, int x, int gc0, float (&v)[32]) {
  const bool full = gc0 + 32 <= p.Cout;
  if (p.bias) {
    if (full) {
      const float4* b4 = reinterpret_cast<const float4*>(p.bias + gc0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(b4 + q);
        v[4 * q] += b.x;
        v[4 * q + 1] += b.y;
        v[4 * q + 2] += b.z;
        v[4 * q + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (gc0 + j < p.Cout) v[j] += __ldg(p.bias + gc0 + j);
    }
  }
  const long long pix = ((long long)t * p.H + y) * p.W + x;
  if (p.mode == 2) {  // RGB8 head: frames in [-1, 1] -> uint8
    uint8_t* o = reinterpret_cast<uint8_t*>(p.out) + pix * p.out_ld;
    for (int j = 0; j < 32 && gc0 + j < p.Cout; ++j) {
      float f = rintf((v[j] + 1.f) * 127.5f);
      f = fminf(fmaxf(f, 0.f), 255.f);
      o[gc0 + j] = (uint8_t)f;
    }
    return;
  }
  long long dst = pix;
  int c0 = gc0;
  if (p.mode == 1) {  // time split: channel block j of width Cout/2 -> output frame 2t + j
    const int half = p.Cout >> 1;
    const int j = gc0 / half;
    c0 = gc0 - j * half;
    dst = ((long long)(2 * t + j) * p.H + y) * p.W + x;
  }
  if (p.resid && p.resid_f32) {
    const float4* r = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.resid) + pix * p.resid_ld + gc0);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 f = r[q];
      v[4 * q] += f.x;
      v[4 * q + 1] += f.y;
      v[4 * q + 2] += f.z;
      v[4 * q + 3] += f.w;
    }
  } else if (p.resid) {
    const __nv_bfloat16* r = p.resid + pix * p.resid_ld + gc0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 w = *reinterpret_cast<const uint4*>(r + 8 * q);
      const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 f = __bfloat1622float2(h2[e]);
        v[8 * q + 2 * e] += f.x;
        v[8 * q + 2 * e + 1] += f.y;
      }
    }
  }
  if (p.out_f32) {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(p.out) + dst * p.out_ld + c0);
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    return;
  }
  __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + dst * p.out_ld + c0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 w;
    w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
    w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
    w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
    w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
    reinterpret_cast<uint4*>(o)[q] = w;
  }
}

// Epilogue of one pixel (thread) over the tile's BN columns: bias / residual / main store
// per 32-column chunk, then (norm_out) a second pass that normalises the pixel's channels.
template <int BN>
__device__ __forceinline__ void conv_epilogue_tile(const ConvParams& p, uint32_t tmem_row, int n_blk, int t, int y,
                                                   int x) {
  const bool live = x < p.W;
  if constexpr (BN <= 96) {
    if (p.norm_out) {   // register-resident: all BN channels of the pixel stay in registers (no read-back)
      float vals[BN];
      float ss = 0.f;
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        if (c * 32 >= p.Cout) break;   // Cout < BN (warp-uniform)
        uint32_t r[32];
        tmem_ld32(tmem_row + c * 32, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (live) {
          conv_epilogue_values(p, t, y, x, c * 32, v);
          if (p.write_main) conv_store(p, t, y, x, c * 32, v);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          ss += v[j] * v[j];
          vals[c * 32 + j] = v[j];
        }
      }
      if (!live) return;
      const float inv = sqrtf((float)p.Cout) / fmaxf(sqrtf(ss), 1e-12f);
      const long long pix = ((long long)t * p.H + y) * p.W + x;
      uint4* o = reinterpret_cast<uint4*>(p.norm_out + pix * p.norm_ld);
#pragma unroll
      for (int q = 0; q < BN / 8; ++q) {
        if (q * 8 >= p.Cout) break;
        float a[8];
        const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.norm_gamma + 8 * q));
        const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.norm_gamma + 8 * q) + 1);
        const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float f = vals[8 * q + e] * inv * gg[e];
          if (p.norm_silu) f = f * fmaf(0.5f, tanh_fast(0.5f * f), 0.5f);
          a[e] = f;
        }
        o[q] = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]), pack_bf16(a[6], a[7]));
      }
      return;
    }
  }
  float ss = 0.f;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    const int gc0 = n_blk * BN + c0;
    if (gc0 >= p.Cout) break;
    uint32_t r[32];
    tmem_ld32(tmem_row + c0, r);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    if (!live) continue;
    if (p.norm_out) {
      conv_epilogue_values(p, t, y, x, gc0, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) ss += v[j] * v[j];
      if (p.write_main) conv_store(p, t, y, x, gc0, v);
    } else {
      conv_epilogue(p, t, y, x, gc0, v);
    }
  }
  if (!p.norm_out) return;
  // every lane stays in the loop: tcgen05.ld is warp-collective (dead pixels only skip memory)
  const float inv = sqrtf((float)p.Cout) / fmaxf(sqrtf(ss), 1e-12f);
  const long long pix = ((long long)t * p.H + y) * p.W + x;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    if (c0 >= p.Cout) break;
    float v[32];
    if (p.write_main && p.out_f32) {  // the values this thread just stored (same-thread read-back)
      if (!live) continue;
      const float4* o = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.out) + pix * p.out_ld + c0);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = o[q];
        v[4 * q] = f.x;
        v[4 * q + 1] = f.y;
        v[4 * q + 2] = f.z;
        v[4 * q + 3] = f.w;
      }
    } else {  // recompute from the accumulator (no residual on this path)
      uint32_t r[32];
      tmem_ld32(tmem_row + c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      if (!live) continue;
      conv_epilogue_values(p, t, y, x, c0, v);
    }
    __nv_bfloat16* o = p.norm_out + pix * p.norm_ld + c0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float a[8];
      const float4 g0 = __ldg(reinterpret_cast<const float4*>(p.norm_gamma + c0 + 8 * q));
      const float4 g1 = __ldg(reinterpret_cast<const float4*>(p.norm_gamma + c0 + 8 * q) + 1);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float f = v[8 * q + e] * inv * gg[e];
        if (p.norm_silu) f = f * fmaf(0.5f, tanh_fast(0.5f * f), 0.5f);   // silu = f * sigmoid(f), one MUFU
        a[e] = f;
      }
      uint4 w;
      w.x = pack_bf16(a[0], a[1]);
      w.y = pack_bf16(a[2], a[3]);
      w.z = pack_bf16(a[4], a[5]);
      w.w = pack_bf16(a[6], a[7]);
      reinterpret_cast<uint4*>(o)[q] = w;
    }
  }
}

template <int BN, int BK>
__global__ void __launch_bounds__(256, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const ConvParams p) {
  using C = ConvCfg<BN, BK>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id(), lane = lane_id();
  const int num_m = p.T * p.H * p.num_xt;
  const int num_n = (p.Cout + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = p.taps * p.kb_per_tap;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
        const int xt = m_blk % p.num_xt;
        const int ty = m_blk / p.num_xt;
        const int t = ty % p.T, y = ty / p.T;  // frames fastest: the 3 input frames a tap row reads stay in L2
        for (int kb = 0; kb < num_kb; ++kb) {
          const int tap = kb / p.kb_per_tap, cb = kb - tap * p.kb_per_tap;
          const int dx = tap % p.KW, dy = (tap / p.KW) % p.KH, dt = tap / (p.KW * p.KH);
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          tma_load_4d(sa, &tmA, &full_bar[stage], cb * BK, xt * 128 + dx - p.pad_w, y + dy - p.pad_h, t + dt + p.t0);
          tma_load_2d(sb, &tmB, &full_bar[stage], tap * p.Cin + cb * BK, n_blk * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // warp-converged MMA issue, one elected lane
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(128, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_bf16_ss_elect(tmem_d, sdesc(sa + k * 32, 16, C::SBO, C::LAYOUT), sdesc(sb + k * 32, 16, C::SBO, C::LAYOUT),
                        idesc, (kb | k) ? 1u : 0u);
          mma_commit_elect(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_elect(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
      const int xt = m_blk % p.num_xt;
      const int ty = m_blk / p.num_xt;
      const int t = ty % p.T, y = ty / p.T;  // frames fastest: the 3 input frames a tap row reads stay in L2
      const int x = xt * 128 + q * 32 + lane;
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      conv_epilogue_tile<BN>(p, tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, n_blk, t, y, x);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

template <int BN, int BK>
static int launch_conv(const void* in, int T_in, const void* w_t, const ConvParams& p, cudaStream_t s) {
  using C = ConvCfg<BN, BK>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "conv smem attribute");
    configured = true;
  }
  CUtensorMap ta, tb;
  {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.H * p.W * p.Cin * 2};
    uint32_t box[4] = {BK, 128, 1, 1};
    int rc = make_tmap_bf16(&ta, in, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  {
    const long long ktot = (long long)p.taps * p.Cin;
    uint64_t dims[2] = {(uint64_t)ktot, (uint64_t)p.Cout};
    uint64_t strides[1] = {(uint64_t)ktot * 2};
    uint32_t box[2] = {BK, BN};
    int rc = make_tmap_bf16(&tb, w_t, 2, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  const int tiles = p.T * p.H * p.num_xt * ((p.Cout + BN - 1) / BN);
  const int grid = tiles < sm_count() ? tiles : sm_count();
  conv_tc_kernel<BN, BK><<<grid, 256, C::SMEM, s>>>(ta, tb, p);
  return check_launch("conv_tc_kernel");
}

// ---------------------------------------------------------------------------------------
// 3x3 (x KT) variant with dx reuse: per (dt, dy, channel block) ONE haloed TMA box of 130
// pixels (x0-1 .. x0+128) feeds the three dx taps as row-shifted smem views (UMMA
// descriptor start + dx*128 B; the 128B-swizzle XOR follows absolute smem address bits, so
// the shifted views need no base offset — verified on B200), cutting
// the A-operand L2 traffic 3x. BK = 64 (SWIZZLE_128B); B holds the three taps' weights.
constexpr int DXR_AROWS = 130;

// BRES: the whole weight tensor (one N block) stays resident in smem, loaded once per CTA;
// the ring stages only the haloed A rows (the RGB head: 16 weight rows x 27 taps x Cin).
constexpr int DXR_BRES_MAX = 96 * 1024;
template <int BN, int BK, bool BRES = false>
struct DxrCfg {
  static constexpr int ROW = BK * 2;                      // bytes per pixel row of a k-block
  static constexpr int A_BYTES = (DXR_AROWS * ROW + 1023) / 1024 * 1024;
  static constexpr int B_TAP = BN * ROW;
  static constexpr int STAGE_BYTES = BRES ? A_BYTES : A_BYTES + 3 * B_TAP;
  static constexpr int RING = (200 * 1024) - (BRES ? DXR_BRES_MAX : 0);
  static constexpr int STAGES = RING / STAGE_BYTES > 8 ? 8 : RING / STAGE_BYTES;
  static constexpr int OFF_BRES = STAGES * STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * BN <= 64) ? 64 : ((2 * BN <= 128) ? 128 : ((2 * BN <= 256) ? 256 : 512));
  static constexpr int SMEM = STAGES * STAGE_BYTES + (BRES ? DXR_BRES_MAX : 0) + 1024 + 256;
  static constexpr uint32_t LAYOUT = (BK == 64) ? 2u : 4u;  // SWIZZLE_128B / SWIZZLE_64B
  static constexpr uint32_t SBO = 8 * ROW;
};


template <int BN, int BK, bool BRES>
__global__ void __launch_bounds__(256, 1)
    conv_dxr_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmTop, const __grid_constant__ CUtensorMap tmBot,
                    const ConvParams p) {
  using C = DxrCfg<BN, BK, BRES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + (BRES ? DXR_BRES_MAX : 0));
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* bres_bar = tempty_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 3);
  uint8_t* bres = smem + C::OFF_BRES;

  const int warp = warp_id(), lane = lane_id();
  const int num_m = p.T * p.H * p.num_xt;
  const int num_n = (p.Cout + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int rows = p.KT * 3;                  // (dt, dy) pairs
  const int num_kb = rows * p.kb_per_tap;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    mbar_init(bres_bar, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      if (BRES) {  // all (kb, dx) weight tiles of the single N block, once
        mbar_arrive_expect_tx(bres_bar, num_kb * 3 * C::B_TAP);
        for (int kb = 0; kb < num_kb; ++kb) {
          const int r = kb / p.kb_per_tap, cb = kb - r * p.kb_per_tap;
          for (int dx = 0; dx < 3; ++dx)
            tma_load_2d(bres + (kb * 3 + dx) * C::B_TAP, &tmB, bres_bar, (r * 3 + dx) * p.Cin + cb * BK, 0);
        }
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
        const int xt = m_blk % p.num_xt;
        const int ty = m_blk / p.num_xt;
        const int t = ty % p.T, y = ty / p.T;  // frames fastest: the 3 input frames a tap row reads stay in L2
        for (int kb = 0; kb < num_kb; ++kb) {
          const int r = kb / p.kb_per_tap, cb = kb - r * p.kb_per_tap;
          const int dy = r % 3, dt = r / 3;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], DXR_AROWS * C::ROW + (BRES ? 0 : 3 * C::B_TAP));
          const int row = y + dy - 1;
          if (p.halo && row < 0)          // neighbour's last row (or zeros at the global edge)
            tma_load_4d(sa, &tmTop, &full_bar[stage], cb * BK, xt * 128 - 1, 0, t + dt + p.t0);
          else if (p.halo && row >= p.H)  // neighbour's first row
            tma_load_4d(sa, &tmBot, &full_bar[stage], cb * BK, xt * 128 - 1, 0, t + dt + p.t0);
          else
            tma_load_4d(sa, &tmA, &full_bar[stage], cb * BK, xt * 128 - 1, row, t + dt + p.t0);
          const int tap0 = (dt * 3 + dy) * 3;
          if (!BRES)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
              tma_load_2d(sb + dx * C::B_TAP, &tmB, &full_bar[stage], (tap0 + dx) * p.Cin + cb * BK, n_blk * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // warp-converged MMA issue, one elected lane
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(128, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      if (BRES) mbar_wait(bres_bar, 0);
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = BRES ? smem_u32(bres) + kb * 3 * C::B_TAP : sa + C::A_BYTES;
#pragma unroll
          for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16_ss_elect(tmem_d, sdesc(sa + dx * C::ROW + k * 32, 16, C::SBO, C::LAYOUT),
                          sdesc(sb + dx * C::B_TAP + k * 32, 16, C::SBO, C::LAYOUT), idesc, (kb | dx | k) ? 1u : 0u);
          mma_commit_elect(&empty_bar[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_elect(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
      const int xt = m_blk % p.num_xt;
      const int ty = m_blk / p.num_xt;
      const int t = ty % p.T, y = ty / p.T;  // frames fastest: the 3 input frames a tap row reads stay in L2
      const int x = xt * 128 + q * 32 + lane;
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      conv_epilogue_tile<BN>(p, tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, n_blk, t, y, x);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

template <int BN, int BK, bool BRES = false>
static int launch_conv_dxr(const void* in, int T_in, const void* w_t, const ConvParams& p, cudaStream_t s,
                           const void* halo_top = nullptr, const void* halo_bot = nullptr) {
  using C = DxrCfg<BN, BK, BRES>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_dxr_kernel<BN, BK, BRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "conv_dxr smem attribute");
    configured = true;
  }
  CUtensorMap ta, tb;
  {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.H * p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ta, in, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  {
    const long long ktot = (long long)p.taps * p.Cin;
    uint64_t dims[2] = {(uint64_t)ktot, (uint64_t)p.Cout};
    uint64_t strides[1] = {(uint64_t)ktot * 2};
    uint32_t box[2] = {BK, BN};
    int rc = make_tmap_bf16(&tb, w_t, 2, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  const int tiles = p.T * p.H * p.num_xt * ((p.Cout + BN - 1) / BN);
  const int grid = tiles < sm_count() ? tiles : sm_count();
  CUtensorMap ttop = ta, tbot = ta;
  if (p.halo) {  // halo rows: [T_in][1][W][Cin] each
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, 1, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ttop, halo_top, 4, dims, strides, box, BK * 2);
    if (!rc) rc = make_tmap_bf16(&tbot, halo_bot, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  conv_dxr_kernel<BN, BK, BRES><<<grid, 256, C::SMEM, s>>>(ta, tb, ttop, tbot, p);
  return check_launch("conv_dxr_kernel");
}


// CTA-pair variant of the dx-reuse conv (cta_group::2): a pair takes two consecutive 128-pixel
// M-tiles (CTA r owns m-tile 2*pm + r) and one UMMA M=256 covers both; each CTA stages its own
// haloed A box and HALF of the Cout rows of the three dx-tap weight tiles, so per CTA the
// weight bytes staged and read per FLOP halve (the single-CTA kernel is bound by shared-memory
// operand bandwidth at BN <= 192). Completions land on the leader's barriers; MMA commits are
// multicast to both CTAs; each CTA drains its own 128 rows of the accumulator.
//
// MSUB = 2 (Cout 96): each CTA owns two 128-pixel M-subtiles that share every weight stage
// (two A boxes, one set of B taps, two accumulators per TMEM buffer), halving the weight
// bytes each SM pulls from L2 per FLOP. At Cout 96 one subtile's MMAs take 48 clk per K=16
// step against ~61 B/clk of A+B operand fill, which outruns the L2->SM feed.
template <int BN, int BK, int MSUB = 1>
struct DxrPairCfg {
  static constexpr int ROW = BK * 2;
  static constexpr int A_BYTES = (DXR_AROWS * ROW + 1023) / 1024 * 1024;
  static constexpr int B_TAP = (BN / 2) * ROW;           // this CTA's half of the Cout rows
  static constexpr int STAGE_BYTES = MSUB * A_BYTES + 3 * B_TAP;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 10 ? 10 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (2 * MSUB * BN <= 128) ? 128 : ((2 * MSUB * BN <= 256) ? 256 : 512);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t LAYOUT = (BK == 64) ? 2u : 4u;
  static constexpr uint32_t SBO = 8 * ROW;
};

template <int BN, int BK, int MSUB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    conv_dxr_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmTop, const __grid_constant__ CUtensorMap tmBot,
                         const ConvParams p) {
  static_assert(2 * MSUB * BN <= 512, "TMEM: two buffers of MSUB accumulators");
  using C = DxrPairCfg<BN, BK, MSUB>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int num_m = p.T * p.H * p.num_xt;
  const int num_pm = (num_m + 2 * MSUB - 1) / (2 * MSUB);
  const int num_n = (p.Cout + BN - 1) / BN;
  const int num_tiles = num_pm * num_n;
  const int rows = p.KT * 3;
  const int num_kb = rows * p.kb_per_tap;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);  // 4 epilogue warps (of the group owning this accumulator) x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
        const int pm = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
        int xt[MSUB], t[MSUB], y[MSUB];
#pragma unroll
        for (int sub = 0; sub < MSUB; ++sub) {
          // m-tile 2*MSUB*pm + 2*sub + rank; a ragged tail recomputes the last tile (not stored)
          const int m_blk = min(2 * MSUB * pm + 2 * sub + (int)rank, num_m - 1);
          xt[sub] = m_blk % p.num_xt;
          const int ty = m_blk / p.num_xt;
          t[sub] = ty % p.T;
          y[sub] = ty / p.T;
        }
        for (int kb = 0; kb < num_kb; ++kb) {
          const int r = kb / p.kb_per_tap, cb = kb - r * p.kb_per_tap;
          const int dy = r % 3, dt = r / 3;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + MSUB * C::A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (MSUB * DXR_AROWS * C::ROW + 3 * C::B_TAP));
#pragma unroll
          for (int sub = 0; sub < MSUB; ++sub) {
            const int row = y[sub] + dy - 1;
            uint8_t* dst = sa + sub * C::A_BYTES;
            if (p.halo && row < 0)
              tma_load_4d_pair(dst, &tmTop, &full_bar[stage], cb * BK, xt[sub] * 128 - 1, 0, t[sub] + dt + p.t0);
            else if (p.halo && row >= p.H)
              tma_load_4d_pair(dst, &tmBot, &full_bar[stage], cb * BK, xt[sub] * 128 - 1, 0, t[sub] + dt + p.t0);
            else
              tma_load_4d_pair(dst, &tmA, &full_bar[stage], cb * BK, xt[sub] * 128 - 1, row, t[sub] + dt + p.t0);
          }
          const int tap0 = (dt * 3 + dy) * 3;
#pragma unroll
          for (int dx = 0; dx < 3; ++dx)
            tma_load_2d_pair(sb + dx * C::B_TAP, &tmB, &full_bar[stage], (tap0 + dx) * p.Cin + cb * BK,
                             n_blk * BN + (int)rank * (BN / 2));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // warp-converged issue on the leader, one elected lane
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(256, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * MSUB * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + MSUB * C::A_BYTES;
#pragma unroll
          for (int sub = 0; sub < MSUB; ++sub)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                mma_bf16_ss_pair_elect(tmem_d + sub * BN,
                                       sdesc(sa + sub * C::A_BYTES + dx * C::ROW + k * 32, 16, C::SBO, C::LAYOUT),
                                       sdesc(sb + dx * C::B_TAP + k * 32, 16, C::SBO, C::LAYOUT), idesc,
                                       (kb | dx | k) ? 1u : 0u);
          mma_commit_pair_elect(&empty_bar[stage], 0x3);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair_elect(&tfull_bar[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    // two epilogue warpgroups take alternate tiles (group g drains accumulator g): the fused
    // norm / fp32 residual epilogue is longer than one tile's mainloop at Cout = 96
    const int q = warp & 3;
    const int eg = (warp - 4) >> 2;
    int it = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++it) {
      if ((it & 1) != eg) continue;
      const int pm = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int sub = 0; sub < MSUB; ++sub) {
        const int m_raw = 2 * MSUB * pm + 2 * sub + (int)rank;
        const int m_blk = min(m_raw, num_m - 1);
        const int xt = m_blk % p.num_xt;
        const int ty = m_blk / p.num_xt;
        const int t = ty % p.T, y = ty / p.T;
        // a recomputed tail tile drains its accumulator without storing (x out of range)
        const int x = m_raw < num_m ? xt * 128 + q * 32 + lane : p.W;
        conv_epilogue_tile<BN>(p, tmem_base + ((uint32_t)(q * 32) << 16) + (acc * MSUB + sub) * BN, n_blk, t, y, x);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty_bar[acc], 0);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
}

template <int BN, int BK, int MSUB = 1>
static int launch_conv_dxr_pair(const void* in, int T_in, const void* w_t, const ConvParams& p, cudaStream_t s,
                                const void* halo_top = nullptr, const void* halo_bot = nullptr) {
  using C = DxrPairCfg<BN, BK, MSUB>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(conv_dxr_pair_kernel<BN, BK, MSUB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "conv_dxr_pair smem attribute");
    configured = true;
  }
  CUtensorMap ta, tb;
  {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.H * p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ta, in, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  {
    const long long ktot = (long long)p.taps * p.Cin;
    uint64_t dims[2] = {(uint64_t)ktot, (uint64_t)p.Cout};
    uint64_t strides[1] = {(uint64_t)ktot * 2};
    uint32_t box[2] = {BK, BN / 2};
    int rc = make_tmap_bf16(&tb, w_t, 2, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  CUtensorMap ttop = ta, tbot = ta;
  if (p.halo) {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, 1, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ttop, halo_top, 4, dims, strides, box, BK * 2);
    if (!rc) rc = make_tmap_bf16(&tbot, halo_bot, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  const int num_m = p.T * p.H * p.num_xt;
  const int tiles = ((num_m + 2 * MSUB - 1) / (2 * MSUB)) * ((p.Cout + BN - 1) / BN);
  const int max_pairs = sm_count() / 2;
  const int pairs = tiles < max_pairs ? tiles : max_pairs;
  conv_dxr_pair_kernel<BN, BK, MSUB><<<2 * pairs, 384, C::SMEM, s>>>(ta, tb, ttop, tbot, p);
  return check_launch("conv_dxr_pair_kernel");
}

// Vertical-reuse pair kernel (Cout 96, BK 32, 3x3 spatial taps): a CTA's two 128-pixel
// M-subtiles are vertically adjacent output rows (y0, y0+1) of one x range, so a stage
// (dt, channel block) stages the 4 input rows y0-1 .. y0+2 once (instead of 3 rows per
// subtile) plus all 9 (dy, dx) weight taps, and subtile s reads input row s + dy for tap dy.
// Operand bytes through the L2->SM fabric per output pixel drop from 3 A rows + half a weight
// set to 2 A rows + half a weight set (the 96-channel convs are bound by that feed).
template <int BN, int BK>
struct DxrVertCfg {
  static constexpr int ROW = BK * 2;
  static constexpr int A_BYTES = (DXR_AROWS * ROW + 1023) / 1024 * 1024;
  static constexpr int B_TAP = (BN / 2) * ROW;
  static constexpr int STAGE_BYTES = 4 * A_BYTES + 9 * B_TAP;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = (4 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr uint32_t LAYOUT = (BK == 64) ? 2u : 4u;
  static constexpr uint32_t SBO = 8 * ROW;
};

template <int BN, int BK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    conv_dxr_vert_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmTop, const __grid_constant__ CUtensorMap tmBot,
                         const ConvParams p) {
  using C = DxrVertCfg<BN, BK>;
  static_assert(C::STAGES >= 2, "stage ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int num_xp = (p.num_xt + 1) / 2;      // x-tile pairs (CTA rank r takes x tile 2*xp + r)
  const int num_yy = (p.H + 1) / 2;           // output row pairs (subtile s takes row 2*yy + s)
  const int num_n = (p.Cout + BN - 1) / BN;
  const int num_tiles = num_xp * p.T * num_yy * num_n;
  const int num_kb = p.KT * p.kb_per_tap;     // stages per tile: (dt, channel block)

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto decode = [&](int tile, int& xt, int& t, int& yy, int& n_blk) {
    n_blk = tile % num_n;
    int r = tile / num_n;
    const int xp = r % num_xp;
    r /= num_xp;
    t = r % p.T;
    yy = r / p.T;
    xt = 2 * xp + (int)rank;
  };

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters) {
        int xt, t, yy, n_blk;
        decode(tile, xt, t, yy, n_blk);
        xt = min(xt, p.num_xt - 1);  // odd x-tile count: the spare CTA recomputes (not stored)
        const int y0 = 2 * yy;
        for (int kb = 0; kb < num_kb; ++kb) {
          const int dt = kb / p.kb_per_tap, cb = kb - dt * p.kb_per_tap;
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + 4 * C::A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * (4 * DXR_AROWS * C::ROW + 9 * C::B_TAP));
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = y0 - 1 + i;
            uint8_t* dst = sa + i * C::A_BYTES;
            if (p.halo && row < 0)
              tma_load_4d_pair(dst, &tmTop, &full_bar[stage], cb * BK, xt * 128 - 1, 0, t + dt + p.t0);
            else if (p.halo && row >= p.H)
              tma_load_4d_pair(dst, &tmBot, &full_bar[stage], cb * BK, xt * 128 - 1, 0, t + dt + p.t0);
            else
              tma_load_4d_pair(dst, &tmA, &full_bar[stage], cb * BK, xt * 128 - 1, row, t + dt + p.t0);
          }
#pragma unroll
          for (int tap = 0; tap < 9; ++tap)   // (dy, dx)
            tma_load_2d_pair(sb + tap * C::B_TAP, &tmB, &full_bar[stage], (dt * 9 + tap) * p.Cin + cb * BK,
                             n_blk * BN + (int)rank * (BN / 2));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(256, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * 2 * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + 4 * C::A_BYTES;
#pragma unroll
          for (int sub = 0; sub < 2; ++sub)
#pragma unroll
            for (int dy = 0; dy < 3; ++dy)
#pragma unroll
              for (int dx = 0; dx < 3; ++dx)
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                  mma_bf16_ss_pair_elect(tmem_d + sub * BN,
                                         sdesc(sa + (sub + dy) * C::A_BYTES + dx * C::ROW + k * 32, 16, C::SBO, C::LAYOUT),
                                         sdesc(sb + (dy * 3 + dx) * C::B_TAP + k * 32, 16, C::SBO, C::LAYOUT), idesc,
                                         (kb | dy | dx | k) ? 1u : 0u);
          mma_commit_pair_elect(&empty_bar[stage], 0x3);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair_elect(&tfull_bar[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int eg = (warp - 4) >> 2;
    int it = 0;
    for (int tile = cluster; tile < num_tiles; tile += n_clusters, ++it) {
      if ((it & 1) != eg) continue;
      int xt, t, yy, n_blk;
      decode(tile, xt, t, yy, n_blk);
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int sub = 0; sub < 2; ++sub) {
        const int y = 2 * yy + sub;
        // spare x tile or a row past an odd H: drain without storing (x out of range)
        const int x = (xt < p.num_xt && y < p.H) ? xt * 128 + q * 32 + lane : p.W;
        conv_epilogue_tile<BN>(p, tmem_base + ((uint32_t)(q * 32) << 16) + (acc * 2 + sub) * BN, n_blk, t,
                               min(y, p.H - 1), x);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty_bar[acc], 0);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<C::TMEM_COLS>(tmem_base);
}

template <int BN, int BK>
static int launch_conv_dxr_vert(const void* in, int T_in, const void* w_t, const ConvParams& p, cudaStream_t s,
                                const void* halo_top = nullptr, const void* halo_bot = nullptr) {
  using C = DxrVertCfg<BN, BK>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(conv_dxr_vert_kernel<BN, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "conv_dxr_vert smem attribute");
    configured = true;
  }
  CUtensorMap ta, tb;
  {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, (uint64_t)p.H, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.H * p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ta, in, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  {
    const long long ktot = (long long)p.taps * p.Cin;
    uint64_t dims[2] = {(uint64_t)ktot, (uint64_t)p.Cout};
    uint64_t strides[1] = {(uint64_t)ktot * 2};
    uint32_t box[2] = {BK, BN / 2};
    int rc = make_tmap_bf16(&tb, w_t, 2, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  CUtensorMap ttop = ta, tbot = ta;
  if (p.halo) {
    uint64_t dims[4] = {(uint64_t)p.Cin, (uint64_t)p.W, 1, (uint64_t)T_in};
    uint64_t strides[3] = {(uint64_t)p.Cin * 2, (uint64_t)p.W * p.Cin * 2, (uint64_t)p.W * p.Cin * 2};
    uint32_t box[4] = {BK, DXR_AROWS, 1, 1};
    int rc = make_tmap_bf16(&ttop, halo_top, 4, dims, strides, box, BK * 2);
    if (!rc) rc = make_tmap_bf16(&tbot, halo_bot, 4, dims, strides, box, BK * 2);
    if (rc) return rc;
  }
  const int tiles = ((p.num_xt + 1) / 2) * p.T * ((p.H + 1) / 2) * ((p.Cout + BN - 1) / BN);
  const int max_pairs = sm_count() / 2;
  const int pairs = tiles < max_pairs ? tiles : max_pairs;
  conv_dxr_vert_kernel<BN, BK><<<2 * pairs, 384, C::SMEM, s>>>(ta, tb, ttop, tbot, p);
  return check_launch("conv_dxr_vert_kernel");
}

}  // namespace ftb

using namespace ftb;

static int conv3d_impl(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in, int32_t H,
                       int32_t W, int32_t Cin, const void* w_t,
                               int32_t Cout, int32_t KT, int32_t KH, int32_t KW, int32_t t0, const float* bias,
                               const void* resid, int64_t resid_ld, void* out, int64_t out_ld, int32_t T_out,
                               int32_t mode, void* stream, const ftb_conv_norm* nrm = nullptr) {
  const bool norm = nrm && nrm->out;
  if (!in || !w_t || (!out && !(norm && !nrm->write_main)) || T_out <= 0 || H <= 0 || W <= 0 || Cin <= 0 || Cout <= 0)
    return set_error(FTB_EINVAL, "conv3d: bad arguments");
  if (norm) {
    if ((mode & 15) != 0) return set_error(FTB_EINVAL, "conv3d: fused norm needs store mode 0");
    if (Cout > 192 || Cout % 32 || !nrm->gamma || (nrm->ld % 8))
      return set_error(FTB_EINVAL, "conv3d: fused norm needs Cout <= 192 (one N tile), Cout % 32 == 0, gamma");
    if (!nrm->write_main && resid) return set_error(FTB_EINVAL, "conv3d: fused norm without main output takes no residual");
  }
  const int out_f32 = (mode >> 4) & 1, resid_f32 = (mode >> 5) & 1;
  // kernel variant of this call (bits 8-10, 0 = auto): 1 per-tap kernel, 2 dx reuse on CTA pairs,
  // 3 dx reuse single-CTA, 4 CTA pairs with one M-subtile per CTA (A/B benchmarks, tests)
  const int variant = (mode >> 8) & 7;
  if (variant > 4) return set_error(FTB_EINVAL, "conv3d: variant (mode bits 8-10) must be 0..4");
  mode &= 15;
  if (Cin % 8) return set_error(FTB_EINVAL, "conv3d: Cin must be a multiple of 8");
  if ((KH != 1 && KH != 3) || (KW != 1 && KW != 3) || KT < 1 || KT > 3)
    return set_error(FTB_EINVAL, "conv3d: kernel must be {1..3} x {1,3} x {1,3}");
  if (t0 < 0 || t0 + T_out - 1 + KT - 1 >= T_in) return set_error(FTB_EINVAL, "conv3d: input frames out of range");
  if (mode != 2 && (Cout % 32)) return set_error(FTB_EINVAL, "conv3d: Cout must be a multiple of 32");
  if (mode == 1 && (Cout % 64)) return set_error(FTB_EINVAL, "conv3d: time-split needs Cout multiple of 64");
  if (resid && (resid_ld % 8)) return set_error(FTB_EINVAL, "conv3d: resid_ld alignment");
  if (mode != 2 && out && (out_ld % 8)) return set_error(FTB_EINVAL, "conv3d: out_ld alignment");
  ConvParams p{};
  p.T = T_out;
  p.H = H;
  p.W = W;
  p.Cin = Cin;
  p.Cout = Cout;
  p.KT = KT;
  p.KH = KH;
  p.KW = KW;
  p.t0 = t0;
  p.pad_h = KH / 2;
  p.pad_w = KW / 2;
  p.num_xt = (W + 127) / 128;
  p.taps = KT * KH * KW;
  p.bias = bias;
  p.resid = reinterpret_cast<const __nv_bfloat16*>(resid);
  p.resid_ld = resid_ld;
  p.out = out;
  p.out_ld = out_ld;
  p.mode = mode;
  p.out_f32 = out_f32;
  p.resid_f32 = resid_f32;
  p.halo = halo_top != nullptr;
  if (norm) {
    p.norm_gamma = nrm->gamma;
    p.norm_out = reinterpret_cast<__nv_bfloat16*>(nrm->out);
    p.norm_ld = nrm->ld;
    p.norm_silu = nrm->silu;
    p.write_main = nrm->write_main;
  }
  if (p.halo && (!halo_bot || KH != 3 || KW != 3 || Cin % 32))
    return set_error(FTB_EINVAL, "conv3d: halo rows need a 3x3 kernel, both halo buffers and Cin % 32 == 0");
  if ((variant != 1 || p.halo) && KH == 3 && KW == 3 && Cin % 32 == 0) {
    cudaStream_t s0 = reinterpret_cast<cudaStream_t>(stream);
    const void *ht = halo_top, *hb = halo_bot;
    // CTA pairs halve each SM's weight traffic (auto for Cout 96 / 192: the smem-bound levels)
    // (Cout 96 / multiples of 192: the smem- and L2-feed-bound levels); variant 4 = pair
    // without the two-subtile weight sharing at Cout 96 (A/B)
    const bool pair = (variant == 2 || variant == 4 || variant == 0) &&
                      (Cout == 96 || Cout % 192 == 0) && !(norm && Cout > 192);
    if (pair) {
      const bool msub = variant != 4;
      if (Cin % 64 == 0) {
        p.kb_per_tap = Cin / 64;
        if (Cout == 96)
          return msub ? launch_conv_dxr_pair<96, 64, 2>(in, T_in, w_t, p, s0, ht, hb)
                      : launch_conv_dxr_pair<96, 64>(in, T_in, w_t, p, s0, ht, hb);
        return launch_conv_dxr_pair<192, 64>(in, T_in, w_t, p, s0, ht, hb);
      }
      p.kb_per_tap = Cin / 32;
      if (Cout == 96 && variant != 2)   // vertical row reuse (variant 2 keeps two x-subtiles)
        return msub ? launch_conv_dxr_vert<96, 32>(in, T_in, w_t, p, s0, ht, hb)
                    : launch_conv_dxr_pair<96, 32>(in, T_in, w_t, p, s0, ht, hb);
      if (Cout == 96)
        return msub ? launch_conv_dxr_pair<96, 32, 2>(in, T_in, w_t, p, s0, ht, hb)
                    : launch_conv_dxr_pair<96, 32>(in, T_in, w_t, p, s0, ht, hb);
      return launch_conv_dxr_pair<192, 32>(in, T_in, w_t, p, s0, ht, hb);
    }
    // Cout <= 16 (the RGB head): 16-row weight boxes; a 32-row box moved 29 zero-filled rows
    // per tap through the L2->SM fabric (11.6 of the head conv's 27 GB)
    if (Cin % 64 == 0) {
      p.kb_per_tap = Cin / 64;
      if (Cout <= 16)
        return (long long)KT * 3 * p.kb_per_tap * 3 * 16 * 128 <= DXR_BRES_MAX
                   ? launch_conv_dxr<16, 64, true>(in, T_in, w_t, p, s0, ht, hb)
                   : launch_conv_dxr<16, 64>(in, T_in, w_t, p, s0, ht, hb);
      if (Cout <= 32) return launch_conv_dxr<32, 64>(in, T_in, w_t, p, s0, ht, hb);
      if (Cout <= 96) return launch_conv_dxr<96, 64>(in, T_in, w_t, p, s0, ht, hb);
      return launch_conv_dxr<192, 64>(in, T_in, w_t, p, s0, ht, hb);
    }
    p.kb_per_tap = Cin / 32;
    if (Cout <= 16)   // weights resident in smem when they fit (the RGB head: 81 KB at Cin 96)
      return (long long)KT * 3 * p.kb_per_tap * 3 * 16 * 64 <= DXR_BRES_MAX
                 ? launch_conv_dxr<16, 32, true>(in, T_in, w_t, p, s0, ht, hb)
                 : launch_conv_dxr<16, 32>(in, T_in, w_t, p, s0, ht, hb);
    if (Cout <= 32) return launch_conv_dxr<32, 32>(in, T_in, w_t, p, s0, ht, hb);
    if (Cout <= 96) return launch_conv_dxr<96, 32>(in, T_in, w_t, p, s0, ht, hb);
    return launch_conv_dxr<192, 32>(in, T_in, w_t, p, s0, ht, hb);
  }
  const bool bk32 = (Cin % 64) != 0 && (Cin % 32) == 0;
  const int BK = (Cin <= 32 || bk32) ? 32 : 64;
  p.kb_per_tap = (Cin + BK - 1) / BK;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int bn = Cout <= 32 ? 32 : (Cout == 96 ? 96 : 192);
  if (Cout > 32 && Cout != 96 && (Cout % 192) && Cout != 64 && Cout != 128)
    ;  // falls through to 192 tiles with a masked tail
  if (BK == 32) {
    if (bn == 32) return launch_conv<32, 32>(in, T_in, w_t, p, s);
    if (bn == 96) return launch_conv<96, 32>(in, T_in, w_t, p, s);
    return launch_conv<192, 32>(in, T_in, w_t, p, s);
  }
  if (bn == 32) return launch_conv<32, 64>(in, T_in, w_t, p, s);
  if (bn == 96) return launch_conv<96, 64>(in, T_in, w_t, p, s);
  return launch_conv<192, 64>(in, T_in, w_t, p, s);
}

extern "C" int ftb_conv3d_bf16(const void* in, int32_t T_in, int32_t H, int32_t W, int32_t Cin, const void* w_t,
                               int32_t Cout, int32_t KT, int32_t KH, int32_t KW, int32_t t0, const float* bias,
                               const void* resid, int64_t resid_ld, void* out, int64_t out_ld, int32_t T_out,
                               int32_t mode, void* stream) {
  return conv3d_impl(in, nullptr, nullptr, T_in, H, W, Cin, w_t, Cout, KT, KH, KW, t0, bias, resid, resid_ld, out,
                     out_ld, T_out, mode, stream);
}

extern "C" int ftb_conv3d_norm_bf16(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in,
                                    int32_t H, int32_t W, int32_t Cin, const void* w_t, int32_t Cout, int32_t KT,
                                    int32_t KH, int32_t KW, int32_t t0, const float* bias, const void* resid,
                                    int64_t resid_ld, void* out, int64_t out_ld, int32_t T_out, int32_t mode,
                                    const ftb_conv_norm* norm, void* stream) {
  if (!norm || !norm->out) return set_error(FTB_EINVAL, "conv3d_norm: norm output required");
  if ((halo_top == nullptr) != (halo_bot == nullptr)) return set_error(FTB_EINVAL, "conv3d_norm: both halos or none");
  return conv3d_impl(in, halo_top, halo_bot, T_in, H, W, Cin, w_t, Cout, KT, KH, KW, t0, bias, resid, resid_ld, out,
                     out_ld, T_out, mode, stream, norm);
}

extern "C" int ftb_conv3d_halo_bf16(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in,
                                    int32_t H, int32_t W, int32_t Cin, const void* w_t, int32_t Cout, int32_t KT,
                                    int32_t KH, int32_t KW, int32_t t0, const float* bias, const void* resid,
                                    int64_t resid_ld, void* out, int64_t out_ld, int32_t T_out, int32_t mode,
                                    void* stream) {
  if (!halo_top || !halo_bot) return set_error(FTB_EINVAL, "conv3d_halo: halo buffers required");
  return conv3d_impl(in, halo_top, halo_bot, T_in, H, W, Cin, w_t, Cout, KT, KH, KW, t0, bias, resid, resid_ld, out,
                     out_ld, T_out, mode, stream);
}

// ============================================================ RGB head as a 1x1 GEMM + 27-tap gather
// The 96 -> 3 head conv (3x3x3, RGB8 store) as an implicit GEMM has N = 3 output channels: its
// MMAs run at a few percent of the tensor rate and restage the haloed input for every tap. Here
// the 27 taps x 3 channels become the M = 81 rows of a GEMM over the input pixels of each frame,
//   Y[t][tap * 3 + c][p] = sum_k W[c][k][tap] x[t][p][k]      (x read once, K = Cin)
// stored tap-major per frame (row n of frame t contiguous over its H*W pixels; one GEMM per frame
// keeps a tile's 81 output rows within a frame's 49 MB instead of 81 rows 18 MB apart, which ran
// 2.3x slower on address translation), and a gather sums each output pixel's 27 shifted taps:
// coalesced 2-byte reads along x, every Y value read by exactly one output pixel. Halo rows
// (split decode) get their own small Y block.
namespace ftb {
__global__ void __launch_bounds__(128) head_gather_rgb8_kernel(const __nv_bfloat16* __restrict__ Y,
                                                               const __nv_bfloat16* __restrict__ Yt,
                                                               const __nv_bfloat16* __restrict__ Yb, long long ldh,
                                                               int H, int W, int t0, const float* __restrict__ bias,
                                                               uint8_t* __restrict__ out) {
  const int x = blockIdx.x * 128 + threadIdx.x, y = blockIdx.y, t = blockIdx.z;
  if (x >= W) return;
  const long long hw = (long long)H * W;
  float acc[3] = {bias ? bias[0] : 0.f, bias ? bias[1] : 0.f, bias ? bias[2] : 0.f};
#pragma unroll
  for (int dt = 0; dt < 3; ++dt) {
    const int tt = t0 + t + dt;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = y + dy - 1;
      const __nv_bfloat16* base;
      long long ld;
      if (yy < 0) {
        if (!Yt) continue;
        base = Yt + (long long)tt * W, ld = ldh;
      } else if (yy >= H) {
        if (!Yb) continue;
        base = Yb + (long long)tt * W, ld = ldh;
      } else {
        base = Y + (long long)tt * 81 * hw + (long long)yy * W, ld = hw;
      }
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int xx = x + dx - 1;
        if (xx < 0 || xx >= W) continue;
        const int tap = (dt * 3 + dy) * 3 + dx;
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += __bfloat162float(base[(long long)(tap * 3 + c) * ld + xx]);
      }
    }
  }
  uint8_t* o = out + (((long long)t * H + y) * W + x) * 3;
#pragma unroll
  for (int c = 0; c < 3; ++c) o[c] = (uint8_t)fminf(fmaxf(rintf((acc[c] + 1.f) * 127.5f), 0.f), 255.f);
}
}  // namespace ftb

extern "C" int ftb_conv3d_head_rgb8(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in,
                                    int32_t H, int32_t W, int32_t Cin, const void* w_taps, const float* bias,
                                    void* y_ws, int64_t y_ws_elems, void* out, int32_t T_out, int32_t t0,
                                    void* stream) {
  if (!in || !w_taps || !y_ws || !out || T_in <= 0 || H <= 0 || W <= 0 || Cin <= 0 || (Cin % 8) || T_out <= 0 ||
      t0 < 0 || t0 + T_out + 2 > T_in || (!halo_top) != (!halo_bot))
    return set_error(FTB_EINVAL, "conv3d_head_rgb8: bad arguments (Cin % 8 == 0, t0 + T_out + 2 <= T_in, both halos)");
  const long long hw = (long long)H * W, npix = (long long)T_in * hw, nh = (long long)T_in * W;
  const long long need = 81 * (npix + (halo_top ? 2 * nh : 0));
  if (y_ws_elems < need) return set_error(FTB_EINVAL, "conv3d_head_rgb8: workspace too small");
  if (hw > 0x7fffffffLL || nh > 0x7fffffffLL) return set_error(FTB_EINVAL, "conv3d_head_rgb8: frame too large");
  __nv_bfloat16* Y = reinterpret_cast<__nv_bfloat16*>(y_ws);
  const __nv_bfloat16* X = reinterpret_cast<const __nv_bfloat16*>(in);
  ftb_epilogue e{};
  e.kind = FTB_EPI_BF16;
  e.ldc = hw;
  int rc;
  // per frame: Y[t] = W_taps . X[t]^T, M = 81 tap-channels (A = w_taps [81][Cin]), N = the frame's pixels
  for (int t = 0; t < T_in; ++t) {
    e.out = Y + (long long)t * 81 * hw;
    if ((rc = ftb_gemm_bf16(w_taps, Cin, 1, 0, X + (long long)t * hw * Cin, Cin, 81, (int32_t)hw, Cin, &e, stream)))
      return rc;
  }
  __nv_bfloat16 *Yt = nullptr, *Yb = nullptr;
  if (halo_top) {
    Yt = Y + 81 * npix;
    Yb = Yt + 81 * nh;
    e.ldc = nh;
    e.out = Yt;
    if ((rc = ftb_gemm_bf16(w_taps, Cin, 1, 0, halo_top, Cin, 81, (int32_t)nh, Cin, &e, stream))) return rc;
    e.out = Yb;
    if ((rc = ftb_gemm_bf16(w_taps, Cin, 1, 0, halo_bot, Cin, 81, (int32_t)nh, Cin, &e, stream))) return rc;
  }
  dim3 grid((W + 127) / 128, H, T_out);
  head_gather_rgb8_kernel<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      Y, Yt, Yb, nh, H, W, t0, bias, reinterpret_cast<uint8_t*>(out));
  return check_launch("head_gather_rgb8_kernel");
}
