// HBM-bound kernels of the wan-mode VAE decoder (channel-last bf16):
// RMS norm (+SiLU) over channels and nearest 2x spatial upsampling.
#include "common.cuh"
#include "ftb_internal.h"

namespace ftb {
// Wan RMS_norm: x / max(||x||_2, eps) * sqrt(C) * gamma, then optional SiLU.
// One warp per pixel (C <= 1024, 8-channel 16-byte vectors).
__global__ void rmsnorm_silu_kernel(const __nv_bfloat16* __restrict__ x, long long n_pix, int C,
                                    const float* __restrict__ gamma, float eps, int silu,
                                    __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int nv = C >> 3;
  for (long long pix = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); pix < n_pix; pix += warps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + pix * C);
    uint4 buf[4];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nv) {
        buf[i] = xr[vi];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&buf[i]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          ss += f.x * f.x + f.y * f.y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = sqrtf((float)C) / fmaxf(sqrtf(ss), eps);
    uint4* yr = reinterpret_cast<uint4*>(y + pix * C);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int vi = lane + 32 * i;
      if (vi < nv) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&buf[i]);
        uint4 w;
        uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(h[e]);
          const int c = vi * 8 + 2 * e;
          float a = f.x * inv * __ldg(gamma + c), b = f.y * inv * __ldg(gamma + c + 1);
          if (silu) {
            a = a / (1.f + __expf(-a));
            b = b / (1.f + __expf(-b));
          }
          wp[e] = pack_bf16(a, b);
        }
        yr[vi] = w;
      }
    }
  }
}

// Nearest 2x spatial upsample: y[t, 2i+a, 2j+b, :] = x[t, i, j, :] (16-byte vectors).
// Nearest 2x spatial upsample, channel-last. blockIdx.y = input row (t, y); each thread reads
// one 16-byte input vector once and writes it to the 2x2 output positions (32-bit index math
// per input vector instead of 64-bit div/mod chains per output vector).
__global__ void upsample2x_kernel(const uint4* __restrict__ x, int H, int W, int cv, uint4* __restrict__ y) {
  const long long ty = blockIdx.y;               // t * H + yi
  const int yi = (int)(ty % H);
  const long long t = ty / H;
  const int n = W * cv;
  const uint4* xr = x + ty * n;
  const long long orow = 2LL * W * cv;           // output row length in vectors
  uint4* y0 = y + ((t * (2 * H) + 2 * yi) * orow);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int xi = i / cv, c = i - xi * cv;
    const uint4 v = xr[i];
    const long long o = 2LL * xi * cv + c;
    y0[o] = v;
    y0[o + cv] = v;
    y0[orow + o] = v;
    y0[orow + o + cv] = v;
  }
}
}  // namespace ftb

using namespace ftb;

extern "C" int ftb_rmsnorm_silu_bf16(const void* x, int64_t n_pix, int32_t C, const float* gamma, float eps,
                                     int32_t silu, void* y, void* stream) {
  if (!x || !y || !gamma || C <= 0 || (C % 8) || C > 1024) return set_error(FTB_EINVAL, "rmsnorm: bad arguments");
  if (n_pix <= 0) return FTB_OK;
  long long blocks = (n_pix + 7) / 8;
  long long cap = (long long)sm_count() * 16;
  rmsnorm_silu_kernel<<<(int)(blocks < cap ? blocks : cap), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (const __nv_bfloat16*)x, n_pix, C, gamma, eps, silu, (__nv_bfloat16*)y);
  return check_launch("rmsnorm_silu_kernel");
}

extern "C" int ftb_upsample2x_bf16(const void* x, int32_t T, int32_t H, int32_t W, int32_t C, void* y, void* stream) {
  if (!x || !y || (C % 8)) return set_error(FTB_EINVAL, "upsample2x: bad arguments");
  if ((long long)T * H * W <= 0) return FTB_OK;
  if ((long long)T * H > 65535) return set_error(FTB_EINVAL, "upsample2x: T * H > 65535");
  const int n = W * (C / 8);
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)((long long)T * H));
  upsample2x_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>((const uint4*)x, H, W, C / 8, (uint4*)y);
  return check_launch("upsample2x_kernel");
}

namespace ftb {
// Sampler latents f32 [T][C][H][W] -> channel-last bf16 [T][H][W][ldy] (first VAE conv input).
__global__ void nchw_to_nhwc_kernel(const float* __restrict__ x, int T, int C, int H, int W,
                                    __nv_bfloat16* __restrict__ y, int ldy) {
  const long long total = (long long)T * H * W * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long r = i;
    const int c = (int)(r % C);
    r /= C;
    const int xx = (int)(r % W);
    r /= W;
    const int yy = (int)(r % H);
    const int t = (int)(r / H);
    y[(((long long)t * H + yy) * W + xx) * ldy + c] = __float2bfloat16_rn(x[(((long long)t * C + c) * H + yy) * W + xx]);
  }
}
}  // namespace ftb

extern "C" int ftb_nchw_to_nhwc_bf16(const float* x, int32_t T, int32_t C, int32_t H, int32_t W, void* y,
                                     int32_t ldy, void* stream) {
  if (!x || !y || ldy < C) return set_error(FTB_EINVAL, "nchw_to_nhwc: bad arguments");
  const long long total = (long long)T * H * W * C;
  if (total <= 0) return FTB_OK;
  long long blocks = (total + 255) / 256, cap = (long long)sm_count() * 8;
  nchw_to_nhwc_kernel<<<(int)(blocks < cap ? blocks : cap), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, T, C, H, W, (__nv_bfloat16*)y, ldy);
  return check_launch("nchw_to_nhwc_kernel");
}

namespace ftb {
// fp32 residual-stream variants: RMS norm (+SiLU) f32 -> bf16, and f32 -> bf16 2x upsample.
__global__ void rmsnorm_silu_f32_kernel(const float* __restrict__ x, long long n_pix, int C,
                                        const float* __restrict__ gamma, float eps, int silu,
                                        __nv_bfloat16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  const int nv = C >> 2;
  for (long long pix = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); pix < n_pix; pix += warps) {
    const float4* xr = reinterpret_cast<const float4*>(x + pix * C);
    float ss = 0.f;
    for (int vi = lane; vi < nv; vi += 32) {
      float4 f = xr[vi];
      ss += f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = sqrtf((float)C) / fmaxf(sqrtf(ss), eps);
    uint2* yr = reinterpret_cast<uint2*>(y + pix * C);
    for (int vi = lane; vi < nv; vi += 32) {
      float4 f = xr[vi];
      const int c = vi * 4;
      float a0 = f.x * inv * __ldg(gamma + c), a1 = f.y * inv * __ldg(gamma + c + 1);
      float a2 = f.z * inv * __ldg(gamma + c + 2), a3 = f.w * inv * __ldg(gamma + c + 3);
      if (silu) {
        a0 = a0 / (1.f + __expf(-a0));
        a1 = a1 / (1.f + __expf(-a1));
        a2 = a2 / (1.f + __expf(-a2));
        a3 = a3 / (1.f + __expf(-a3));
      }
      yr[vi] = make_uint2(pack_bf16(a0, a1), pack_bf16(a2, a3));
    }
  }
}

// fp32 -> bf16 variant of upsample2x_kernel (one float4 read, four 8-byte writes).
__global__ void upsample2x_f32_kernel(const float4* __restrict__ x, int H, int W, int cv, uint2* __restrict__ y) {
  const long long ty = blockIdx.y;
  const int yi = (int)(ty % H);
  const long long t = ty / H;
  const int n = W * cv;
  const float4* xr = x + ty * n;
  const long long orow = 2LL * W * cv;
  uint2* y0 = y + ((t * (2 * H) + 2 * yi) * orow);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int xi = i / cv, c = i - xi * cv;
    const float4 f = xr[i];
    const uint2 v = make_uint2(pack_bf16(f.x, f.y), pack_bf16(f.z, f.w));
    const long long o = 2LL * xi * cv + c;
    y0[o] = v;
    y0[o + cv] = v;
    y0[orow + o] = v;
    y0[orow + o + cv] = v;
  }
}
// Decoder mid-block attention helpers. Row softmax: one CTA per score row (fp32 in, bf16 P
// out), three passes over the row (max, sum, write) that re-read it from L1/L2.
__global__ void __launch_bounds__(256) softmax_rows_bf16_kernel(const float* __restrict__ s, long long ld_s, int cols,
                                                                float scale, __nv_bfloat16* __restrict__ p,
                                                                long long ld_p) {
  __shared__ float red[8];
  const float* row = s + (long long)blockIdx.x * ld_s;
  __nv_bfloat16* out = p + (long long)blockIdx.x * ld_p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < cols; j += 256) mx = fmaxf(mx, row[j]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < cols; j += 256) sum += __expf((row[j] - mx) * scale);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float inv = 1.f / tot;
  for (int j = threadIdx.x; j < cols; j += 256) out[j] = __float2bfloat16_rn(__expf((row[j] - mx) * scale) * inv);
}

// 32 x 32 tiles through shared memory (padded against bank conflicts).
__global__ void __launch_bounds__(256) transpose_bf16_kernel(const __nv_bfloat16* __restrict__ x, long long ld_x,
                                                             int rows, int cols, __nv_bfloat16* __restrict__ y,
                                                             long long ld_y) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8)
    if (r0 + i < rows && c0 + tx < cols) tile[i][tx] = x[(long long)(r0 + i) * ld_x + c0 + tx];
  __syncthreads();
  for (int i = ty; i < 32; i += 8)
    if (c0 + i < cols && r0 + tx < rows) y[(long long)(c0 + i) * ld_y + r0 + tx] = tile[tx][i];
}

}  // namespace ftb

extern "C" int ftb_softmax_rows_bf16(const float* s, int64_t ld_s, int32_t rows, int32_t cols, float scale, void* p,
                                     int64_t ld_p, void* stream) {
  if (!s || !p || rows < 0 || cols <= 0 || ld_s < cols || ld_p < cols)
    return set_error(FTB_EINVAL, "softmax_rows: bad arguments");
  if (rows == 0) return FTB_OK;
  softmax_rows_bf16_kernel<<<rows, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      s, ld_s, cols, scale, static_cast<__nv_bfloat16*>(p), ld_p);
  return check_launch("softmax_rows_bf16_kernel");
}

extern "C" int ftb_transpose_bf16(const void* x, int64_t ld_x, int32_t rows, int32_t cols, void* y, int64_t ld_y,
                                  void* stream) {
  if (!x || !y || rows < 0 || cols < 0 || ld_x < cols || ld_y < rows)
    return set_error(FTB_EINVAL, "transpose: bad arguments");
  if (rows == 0 || cols == 0) return FTB_OK;
  dim3 grid((cols + 31) / 32, (rows + 31) / 32);
  transpose_bf16_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), ld_x, rows, cols, static_cast<__nv_bfloat16*>(y), ld_y);
  return check_launch("transpose_bf16_kernel");
}

extern "C" int ftb_rmsnorm_silu_f32(const float* x, int64_t n_pix, int32_t C, const float* gamma, float eps,
                                    int32_t silu, void* y, void* stream) {
  if (!x || !y || !gamma || C <= 0 || (C % 4)) return set_error(FTB_EINVAL, "rmsnorm_f32: bad arguments");
  if (n_pix <= 0) return FTB_OK;
  long long blocks = (n_pix + 7) / 8, cap = (long long)sm_count() * 16;
  rmsnorm_silu_f32_kernel<<<(int)(blocks < cap ? blocks : cap), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      x, n_pix, C, gamma, eps, silu, (__nv_bfloat16*)y);
  return check_launch("rmsnorm_silu_f32_kernel");
}

extern "C" int ftb_upsample2x_f32_bf16(const float* x, int32_t T, int32_t H, int32_t W, int32_t C, void* y,
                                       void* stream) {
  if (!x || !y || (C % 4)) return set_error(FTB_EINVAL, "upsample2x_f32: bad arguments");
  if ((long long)T * H * W <= 0) return FTB_OK;
  if ((long long)T * H > 65535) return set_error(FTB_EINVAL, "upsample2x_f32: T * H > 65535");
  const int n = W * (C / 4);
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)((long long)T * H));
  upsample2x_f32_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>((const float4*)x, H, W, C / 4,
                                                                                  (uint2*)y);
  return check_launch("upsample2x_f32_kernel");
}
