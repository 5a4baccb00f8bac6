// HBM-bound kernels of the denoise step: norm + AdaLN modulation, composite
// assembly / patchify, unpatchify + DDIM update, codec decode, casts, fills.
// All are row- or element-parallel with vectorised, coalesced access; grids
// are sized in multiples of the SM count.
#include <algorithm>

#include "common.cuh"
#include "ftb_internal.h"

namespace ftb {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int THREADS>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < THREADS / 32; ++i) t += red[i];
  return t;
}

// One CTA per row; two-pass mean / population variance in fp32 (LN of
// backends/reference.py:41-46, eps inside the sqrt), then affine / AdaLN
// modulation and a bf16 store.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) norm_modulate_kernel(
    const float* __restrict__ x, long long ldx, int N, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ scale, const float* __restrict__ shift,
    long long mod_ld, int rows_per_group, long long row_offset, float eps, __nv_bfloat16* __restrict__ y,
    long long ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  __shared__ float red[THREADS / 32];
  const long long row = blockIdx.x;
  const float* xr = x + row * ldx;
  float s = 0.f;
  for (int c = threadIdx.x; c < N; c += THREADS) s += xr[c];
  const float mean = block_sum<THREADS>(s, red) / N;
  float ss = 0.f;
  for (int c = threadIdx.x; c < N; c += THREADS) {
    float d = xr[c] - mean;
    ss += d * d;
  }
  const float var = block_sum<THREADS>(ss, red) / N;
  const float rstd = rsqrtf(var + eps);
  const long long g = rows_per_group > 0 ? (row + row_offset) / rows_per_group : 0;
  const float* sc = scale ? scale + g * mod_ld : nullptr;
  const float* sh = shift ? shift + g * mod_ld : nullptr;
  __nv_bfloat16* yr = y + row * ldy;
  for (int c = threadIdx.x; c < N; c += THREADS) {
    float v = (xr[c] - mean) * rstd;
    if (gamma) v *= gamma[c];
    if (sc) v *= 1.f + sc[c];
    if (beta) v += beta[c];
    if (sh) v += sh[c];
    yr[c] = __float2bfloat16_rn(v);
  }
  if (threadIdx.x == 0) {
    if (mean_out) mean_out[row] = mean;
    if (rstd_out) rstd_out[row] = rstd;
  }
}

// Register-resident variant (N % 4 == 0, N <= 4*T*VMAX, 16-byte aligned rows): the
// row is read from HBM once as float4, both passes run on registers, and the output
// leaves as bf16x4. Same arithmetic as norm_modulate_kernel (two-pass fp32).
template <int VMAX, int T, bool STREAM>
__global__ void __launch_bounds__(T) norm_modulate_vec_kernel(
    const float* __restrict__ x, long long ldx, int N, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ scale, const float* __restrict__ shift,
    long long mod_ld, int rows_per_group, long long row_offset, float eps, __nv_bfloat16* __restrict__ y,
    long long ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  __shared__ float red[T / 32];
  const long long row = blockIdx.x;
  const int n4 = N >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + row * ldx);
  float4 v[VMAX];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < VMAX; ++i) {
    const int c = threadIdx.x + i * T;
    v[i] = c < n4 ? (STREAM ? __ldcs(xr + c) : __ldg(xr + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mean = block_sum<T>(s, red) / N;
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VMAX; ++i) {
    if (threadIdx.x + i * T < n4) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      ss += (a * a + b * b) + (c * c + d * d);
    }
  }
  const float rstd = rsqrtf(block_sum<T>(ss, red) / N + eps);
  const long long g = rows_per_group > 0 ? (row + row_offset) / rows_per_group : 0;
  const float4* sc = scale ? reinterpret_cast<const float4*>(scale + g * mod_ld) : nullptr;
  const float4* sh = shift ? reinterpret_cast<const float4*>(shift + g * mod_ld) : nullptr;
  const float4* ga = reinterpret_cast<const float4*>(gamma);
  const float4* be = reinterpret_cast<const float4*>(beta);
  uint2* yr = reinterpret_cast<uint2*>(y + row * ldy);
#pragma unroll
  for (int i = 0; i < VMAX; ++i) {
    const int c = threadIdx.x + i * T;
    if (c < n4) {
      float4 o = make_float4((v[i].x - mean) * rstd, (v[i].y - mean) * rstd, (v[i].z - mean) * rstd,
                             (v[i].w - mean) * rstd);
      if (gamma) {
        const float4 t = __ldg(ga + c);
        o = make_float4(o.x * t.x, o.y * t.y, o.z * t.z, o.w * t.w);
      }
      if (sc) {
        const float4 t = __ldg(sc + c);
        o = make_float4(o.x * (1.f + t.x), o.y * (1.f + t.y), o.z * (1.f + t.z), o.w * (1.f + t.w));
      }
      if (beta) {
        const float4 t = __ldg(be + c);
        o = make_float4(o.x + t.x, o.y + t.y, o.z + t.z, o.w + t.w);
      }
      if (sh) {
        const float4 t = __ldg(sh + c);
        o = make_float4(o.x + t.x, o.y + t.y, o.z + t.z, o.w + t.w);
      }
      yr[c] = make_uint2(pack_bf16(o.x, o.y), pack_bf16(o.z, o.w));
    }
  }
  if (threadIdx.x == 0) {
    if (mean_out) mean_out[row] = mean;
    if (rstd_out) rstd_out[row] = rstd;
  }
}



// Persistent row-range LayerNorm / AdaLN (the default path for 16-byte aligned rows with
// N % (4*T) == 0): each CTA owns a contiguous range of rows and streams them through a ring of
// NS shared-memory slots filled by 1-D TMA bulk copies, so NS rows per CTA are in flight without
// holding registers. The CTA keeps its slice of the modulation — mul = gamma * (1 + scale),
// add = beta + shift of the row's frame group — in registers and reloads it only when the group
// changes (a range spans at most a few groups), instead of re-reading both vectors from L2 for
// every row. Two-pass fp32 statistics per row as above.
template <int V, int T, int NS>
__global__ void __launch_bounds__(T) norm_rows_kernel(
    const float* __restrict__ x, long long ldx, int N, int M, int rows_per_cta, const float* __restrict__ gamma,
    const float* __restrict__ beta, const float* __restrict__ scale, const float* __restrict__ shift,
    long long mod_ld, int rows_per_group, long long row_offset, float eps, __nv_bfloat16* __restrict__ y,
    long long ldy, float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  extern __shared__ __align__(128) uint8_t norm_sm[];
  __shared__ float red[T / 32];
  float4* ring = reinterpret_cast<float4*>(norm_sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(norm_sm + (size_t)NS * N * 4);
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(M, r0 + rows_per_cta);
  if (r0 >= r1) return;
  const uint32_t row_bytes = (uint32_t)N * 4;
  const int n4 = N >> 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < NS && r0 + s < r1; ++s) {
      mbar_arrive_expect_tx(&full[s], row_bytes);
      bulk_load_1d(ring + (size_t)s * n4, x + (long long)(r0 + s) * ldx, row_bytes, &full[s]);
    }
  long long gcur = -1;
  float4 mul[V], add[V];
  for (int r = r0, it = 0; r < r1; ++r, ++it) {
    const long long g = rows_per_group > 0 ? (r + row_offset) / rows_per_group : 0;
    if (g != gcur) {   // CTA-uniform
      gcur = g;
      const float4* sc = scale ? reinterpret_cast<const float4*>(scale + g * mod_ld) : nullptr;
      const float4* sh = shift ? reinterpret_cast<const float4*>(shift + g * mod_ld) : nullptr;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int c = threadIdx.x + i * T;
        float4 m = gamma ? __ldg(reinterpret_cast<const float4*>(gamma) + c) : make_float4(1.f, 1.f, 1.f, 1.f);
        float4 a = beta ? __ldg(reinterpret_cast<const float4*>(beta) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (sc) {
          const float4 t = __ldg(sc + c);
          m = make_float4(m.x * (1.f + t.x), m.y * (1.f + t.y), m.z * (1.f + t.z), m.w * (1.f + t.w));
        }
        if (sh) {
          const float4 t = __ldg(sh + c);
          a = make_float4(a.x + t.x, a.y + t.y, a.z + t.z, a.w + t.w);
        }
        mul[i] = m;
        add[i] = a;
      }
    }
    const int slot = it % NS;
    mbar_wait(&full[slot], (uint32_t)(it / NS) & 1);
    float4 v[V];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      v[i] = ring[(size_t)slot * n4 + threadIdx.x + i * T];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    const float mean = block_sum<T>(s, red) / N;
    // every thread has read the slot (block_sum's barriers): refill it NS rows ahead
    if (threadIdx.x == 0 && r + NS < r1) {
      mbar_arrive_expect_tx(&full[slot], row_bytes);
      bulk_load_1d(ring + (size_t)slot * n4, x + (long long)(r + NS) * ldx, row_bytes, &full[slot]);
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
      ss += (a * a + b * b) + (c * c + d * d);
    }
    const float rstd = rsqrtf(block_sum<T>(ss, red) / N + eps);
    uint2* yr = reinterpret_cast<uint2*>(y + (long long)r * ldy);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float4 m = mul[i], a = add[i];
      const float ox = fmaf((v[i].x - mean) * rstd, m.x, a.x), oy = fmaf((v[i].y - mean) * rstd, m.y, a.y);
      const float oz = fmaf((v[i].z - mean) * rstd, m.z, a.z), ow = fmaf((v[i].w - mean) * rstd, m.w, a.w);
      yr[threadIdx.x + i * T] = make_uint2(pack_bf16(ox, oy), pack_bf16(oz, ow));
    }
    if (threadIdx.x == 0) {
      if (mean_out) mean_out[r] = mean;
      if (rstd_out) rstd_out[r] = rstd;
    }
  }
}

// Composite assembly (diffusion.py:150-179 + stacked :133-135) fused with the
// 2x2 spatial patchify of the wan-mode token grid. One thread per output element.
__global__ void patchify_kernel(const float* __restrict__ motion, const float* __restrict__ z,
                                const float* __restrict__ ref, int Lm, int Lc, int D, int H, int W, int ph, int pw,
                                __nv_bfloat16* __restrict__ out, long long ldo, long long total) {
  const int gh = H / ph, gw = W / pw;
  const long long tpf = (long long)gh * gw;
  const int C = 2 * D + 1;
  const int F = C * ph * pw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long tok = i / ldo;
    const int feat = (int)(i - tok * ldo);
    float v = 0.f;
    if (feat < F) {
      const int f = (int)(tok / tpf);
      const int rem = (int)(tok - f * tpf);
      const int ty = rem / gw, tx = rem - (rem / gw) * gw;
      const int c = feat / (ph * pw);
      const int pr = feat - c * ph * pw;
      const int py = pr / pw, px = pr - (pr / pw) * pw;
      const int yy = ty * ph + py, xx = tx * pw + px;
      const long long pix = (long long)yy * W + xx;
      if (c < D) {
        v = (f < Lm) ? motion[((long long)f * D + c) * H * W + pix] : z[((long long)(f - Lm) * D + c) * H * W + pix];
      } else if (c == D) {
        v = (f == 0) ? 1.f : 0.f;  // z_mask = [1, 0, ...]
      } else {
        v = (f == 0) ? ref[(long long)(c - D - 1) * H * W + pix] : 0.f;  // z_cond row 0 = reference
      }
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// Patchify of an arbitrary stacked composite [Lc][C][H][W] (the caller's own z_mask / z_cond
// rows: any CompositeInput the reference's Denoiser.forward accepts, net.py:223-238).
__global__ void patchify_stacked_kernel(const float* __restrict__ st, int Lc, int C, int H, int W, int ph, int pw,
                                        __nv_bfloat16* __restrict__ out, long long ldo, long long total) {
  const int gh = H / ph, gw = W / pw;
  const long long tpf = (long long)gh * gw;
  const int F = C * ph * pw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long tok = i / ldo;
    const int feat = (int)(i - tok * ldo);
    float v = 0.f;
    if (feat < F) {
      const int f = (int)(tok / tpf);
      const int rem = (int)(tok - f * tpf);
      const int ty = rem / gw, tx = rem - (rem / gw) * gw;
      const int c = feat / (ph * pw);
      const int pr = feat - c * ph * pw;
      const int py = pr / pw, px = pr - (pr / pw) * pw;
      v = st[(((long long)f * C + c) * H + ty * ph + py) * W + tx * pw + px];
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// x0 tokens -> target-frame latents; DDIM update of the sampler state
// (diffusion.py:229-236): eps = (z - a_i x0)/s_i ; z = a_n x0 + s_n eps.
__global__ void unpatch_ddim_kernel(const float* __restrict__ x0t, long long ldx, int Lm, int Lc, int D, int H,
                                    int W, int ph, int pw, float* __restrict__ z, float* __restrict__ x0_out,
                                    float a_i, float s_i, float a_n, float s_n, int update, long long total) {
  const int gh = H / ph, gw = W / pw;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    // i indexes x0_out [(Lc-Lm)][D][H][W]
    long long t = i;
    const int xx = (int)(t % W);
    t /= W;
    const int yy = (int)(t % H);
    t /= H;
    const int c = (int)(t % D);
    const int ft = (int)(t / D);
    const int f = ft + Lm;
    const int ty = yy / ph, py = yy - ty * ph, tx = xx / pw, px = xx - tx * pw;
    const long long tok = (long long)f * gh * gw + (long long)ty * gw + tx;
    const float x0 = x0t[tok * ldx + (c * ph + py) * pw + px];
    x0_out[i] = x0;
    if (update) {
      const float zi = z[i];
      const float eps = (zi - a_i * x0) / s_i;
      z[i] = a_n * x0 + s_n * eps;
    }
  }
}

__global__ void codec_decode_kernel(const float* __restrict__ lat, const float* __restrict__ Q,
                                    float* __restrict__ out, int n, int D) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * D) return;
  const int r = i / D, c = i - (i / D) * D;
  float acc = 0.f;
  for (int k = 0; k < D; ++k) acc += lat[r * D + k] * Q[k * D + c];
  out[i] = acc;
}

__global__ void gelu_bf16_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(gelu_tanh(__bfloat162float(x[i])));
}
__global__ void silu_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float v = x[i];
    y[i] = __float2bfloat16_rn(v / (1.f + __expf(-v)));
  }
}
__global__ void cast_f2b_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}
__global__ void cast_b2f_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __bfloat162float(x[i]);
}

// Counter-based normal: splitmix64 hash of (seed, index) -> two uniforms -> Box-Muller.
__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ float normal_at(uint64_t seed, long long i) {
  uint64_t h = splitmix(seed ^ splitmix((uint64_t)i));
  float u1 = ((uint32_t)(h >> 40) + 1) * (1.0f / 16777217.0f);
  float u2 = ((uint32_t)(h & 0xFFFFFF)) * (1.0f / 16777216.0f);
  return sqrtf(-2.f * __logf(u1)) * __cosf(6.28318530718f * u2);
}
__global__ void fill_normal_bf16_kernel(__nv_bfloat16* out, long long n, uint64_t seed, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(normal_at(seed, i) * scale);
}
__global__ void fill_normal_f32_kernel(float* out, long long n, uint64_t seed, float scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = normal_at(seed, i) * scale;
}
__global__ void count_nonfinite_kernel(const float* __restrict__ x, long long n, int* out) {
  int c = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    c += !isfinite(x[i]);
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// out[l][f][j] = a[f][j] + b[l][j]  (per-frame AdaLN vectors + per-layer learned offsets)
__global__ void add_bcast_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                                 long long F, long long n, long long total) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long j = i % n;
    const long long lf = i / n;
    const long long f = lf % F, l = lf / F;
    out[i] = a[f * n + j] + b[l * n + j];
  }
}

static inline int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  long long cap = (long long)sm_count() * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace ftb

using namespace ftb;
#define S(stream) reinterpret_cast<cudaStream_t>(stream)

extern "C" int ftb_norm_modulate(const float* x, int64_t ldx, int32_t M, int32_t N, const float* gamma,
                                 const float* beta, const float* scale, const float* shift, int64_t mod_ld,
                                 int32_t rows_per_group, int64_t row_offset, float eps, void* y, int64_t ldy,
                                 float* mean_out, float* rstd_out, void* stream) {
  if (!x || !y || M < 0 || N <= 0) return set_error(FTB_EINVAL, "norm: bad arguments");
  if (M == 0) return FTB_OK;
  if ((scale || shift) && rows_per_group <= 0) return set_error(FTB_EINVAL, "norm: modulation needs rows_per_group");
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = (N % 4 == 0) && N <= 4 * 256 * 8 && (ldx % 4 == 0) && (ldy % 4 == 0) && (!scale || mod_ld % 4 == 0) &&
                   al16(x) && (reinterpret_cast<uintptr_t>(y) & 7) == 0 && (!gamma || al16(gamma)) &&
                   (!beta || al16(beta)) && (!scale || al16(scale)) && (!shift || al16(shift)) && N >= 512;
  // persistent TMA-ring kernel: whole float4 slices per thread, 16-byte aligned rows
  {
    const int n4 = N / 4;
    const int T = (n4 % 256 == 0 && n4 / 256 <= 8) ? 256 : ((n4 % 128 == 0 && n4 / 128 <= 8) ? 128 : 0);
    constexpr int NS = 4;
    const size_t smem = (size_t)NS * N * 4 + NS * 8;
    if (vec && T && ((ldx * 4) % 16 == 0) && smem <= 110 * 1024) {
      const int V = n4 / T;
      // CTAs per SM: as many rings as ~200 KB of shared memory holds (2 at m = 5120: 80 KB rings,
      // 8 at m = 1536), so 8-16 rows per SM are in flight
      const int cps = (int)std::min<size_t>(8, std::max<size_t>(1, (200 * 1024) / smem));
      const int grid0 = sm_count() * cps;
      const int grid = M < grid0 ? M : grid0;
      const int rpc = (M + grid - 1) / grid;
#define FTB_NORM_ROWS(VV, TT)                                                                                        \
  do {                                                                                                                \
    static bool cfg_done = false;                                                                                     \
    if (!cfg_done) {                                                                                                  \
      cudaFuncSetAttribute(norm_rows_kernel<VV, TT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);    \
      cfg_done = true;                                                                                                \
    }                                                                                                                 \
    norm_rows_kernel<VV, TT, NS><<<grid, TT, smem, S(stream)>>>(x, ldx, N, M, rpc, gamma, beta, scale, shift, mod_ld, \
                                                                rows_per_group, row_offset, eps, (__nv_bfloat16*)y,   \
                                                                ldy, mean_out, rstd_out);                             \
  } while (0)
      if (T == 256) {
        switch (V) {
          case 1: FTB_NORM_ROWS(1, 256); break;
          case 2: FTB_NORM_ROWS(2, 256); break;
          case 3: FTB_NORM_ROWS(3, 256); break;
          case 4: FTB_NORM_ROWS(4, 256); break;
          case 5: FTB_NORM_ROWS(5, 256); break;
          case 6: FTB_NORM_ROWS(6, 256); break;
          case 7: FTB_NORM_ROWS(7, 256); break;
          default: FTB_NORM_ROWS(8, 256); break;
        }
      } else {
        switch (V) {
          case 1: FTB_NORM_ROWS(1, 128); break;
          case 2: FTB_NORM_ROWS(2, 128); break;
          case 3: FTB_NORM_ROWS(3, 128); break;
          case 4: FTB_NORM_ROWS(4, 128); break;
          case 5: FTB_NORM_ROWS(5, 128); break;
          case 6: FTB_NORM_ROWS(6, 128); break;
          case 7: FTB_NORM_ROWS(7, 128); break;
          default: FTB_NORM_ROWS(8, 128); break;
        }
      }
#undef FTB_NORM_ROWS
      return check_launch("norm_rows_kernel");
    }
  }
  const bool narrow = N <= 4 * 128 * 4;
  if (vec && narrow && (N / 4) % 128 == 0) {
    // narrow rows (1.3B: m = 1536): 128 threads x 3 float4, every lane busy, twice the rows
    // resident per SM (at 256 threads half the lanes idled in the second float4)
    const int nv = N / 4 / 128;
#define FTB_NORM_VEC128(V)                                                                                          \
  norm_modulate_vec_kernel<V, 128, true><<<M, 128, 0, S(stream)>>>(x, ldx, N, gamma, beta, scale, shift, mod_ld, \
                                                                   rows_per_group, row_offset, eps,              \
                                                                   (__nv_bfloat16*)y, ldy, mean_out, rstd_out)
    if (nv <= 2)
      FTB_NORM_VEC128(2);
    else if (nv <= 3)
      FTB_NORM_VEC128(3);
    else
      FTB_NORM_VEC128(4);
#undef FTB_NORM_VEC128
  } else if (vec) {
    const int nv = (N / 4 + 255) / 256;   // float4 per thread at 256 threads
#define FTB_NORM_VEC(V)                                                                                             \
  norm_modulate_vec_kernel<V, 256, true><<<M, 256, 0, S(stream)>>>(x, ldx, N, gamma, beta, scale, shift, mod_ld, \
                                                                   rows_per_group, row_offset, eps,              \
                                                                   (__nv_bfloat16*)y, ldy, mean_out, rstd_out)
    if (nv <= 2)
      FTB_NORM_VEC(2);
    else if (nv <= 4)
      FTB_NORM_VEC(4);
    else if (nv <= 5)
      FTB_NORM_VEC(5);
    else
      FTB_NORM_VEC(8);
#undef FTB_NORM_VEC
  } else if (N >= 1024)
    norm_modulate_kernel<256><<<M, 256, 0, S(stream)>>>(x, ldx, N, gamma, beta, scale, shift, mod_ld, rows_per_group,
                                                          row_offset, eps, (__nv_bfloat16*)y, ldy, mean_out, rstd_out);
  else
    norm_modulate_kernel<32><<<M, 32, 0, S(stream)>>>(x, ldx, N, gamma, beta, scale, shift, mod_ld, rows_per_group,
                                                        row_offset, eps, (__nv_bfloat16*)y, ldy, mean_out, rstd_out);
  return check_launch("norm_modulate_kernel");
}

extern "C" int ftb_patchify_composite(const float* motion, const float* z, const float* reference, int32_t Lm,
                                      int32_t Lc, int32_t D, int32_t H, int32_t W, int32_t ph, int32_t pw, void* out,
                                      int64_t ldo, void* stream) {
  if (!z || !reference || !out || Lc <= Lm || Lm < 0 || D <= 0 || H % ph || W % pw)
    return set_error(FTB_EINVAL, "patchify: bad arguments");
  if (Lm > 0 && !motion) return set_error(FTB_EINVAL, "patchify: motion required");
  if (ldo < (int64_t)(2 * D + 1) * ph * pw) return set_error(FTB_EINVAL, "patchify: ldo too small");
  long long tokens = (long long)Lc * (H / ph) * (W / pw);
  long long total = tokens * ldo;
  patchify_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(motion, z, reference, Lm, Lc, D, H, W, ph, pw,
                                                               (__nv_bfloat16*)out, ldo, total);
  return check_launch("patchify_kernel");
}

extern "C" int ftb_patchify_stacked(const float* stacked, int32_t Lc, int32_t C, int32_t H, int32_t W, int32_t ph,
                                    int32_t pw, void* out, int64_t ldo, void* stream) {
  if (!stacked || !out || Lc <= 0 || C <= 0 || ph <= 0 || pw <= 0 || H % ph || W % pw)
    return set_error(FTB_EINVAL, "patchify_stacked: bad arguments");
  if (ldo < (int64_t)C * ph * pw) return set_error(FTB_EINVAL, "patchify_stacked: ldo too small");
  const long long total = (long long)Lc * (H / ph) * (W / pw) * ldo;
  patchify_stacked_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(stacked, Lc, C, H, W, ph, pw,
                                                                      (__nv_bfloat16*)out, ldo, total);
  return check_launch("patchify_stacked_kernel");
}

extern "C" int ftb_unpatch_ddim(const float* x0_tok, int64_t ldx, int32_t Lm, int32_t Lc, int32_t D, int32_t H,
                                int32_t W, int32_t ph, int32_t pw, float* z, float* x0_out, float a_i, float s_i,
                                float a_n, float s_n, int32_t update, void* stream) {
  if (!x0_tok || !x0_out || Lc <= Lm || H % ph || W % pw) return set_error(FTB_EINVAL, "unpatch: bad arguments");
  if (update && (!z || s_i == 0.f)) return set_error(FTB_EINVAL, "unpatch: DDIM update needs z and sigma > 0");
  long long total = (long long)(Lc - Lm) * D * H * W;
  unpatch_ddim_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(x0_tok, ldx, Lm, Lc, D, H, W, ph, pw, z, x0_out,
                                                                   a_i, s_i, a_n, s_n, update, total);
  return check_launch("unpatch_ddim_kernel");
}

extern "C" int ftb_codec_decode(const float* latents, const float* Q, float* frames, int32_t n, int32_t D,
                                void* stream) {
  if (!latents || !Q || !frames || n < 0 || D <= 0) return set_error(FTB_EINVAL, "codec: bad arguments");
  if (n == 0) return FTB_OK;
  codec_decode_kernel<<<(n * D + 127) / 128, 128, 0, S(stream)>>>(latents, Q, frames, n, D);
  return check_launch("codec_decode_kernel");
}

extern "C" int ftb_gelu_bf16(const void* x, void* y, int64_t n, void* stream) {
  if (n <= 0) return FTB_OK;
  gelu_bf16_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>((const __nv_bfloat16*)x, (__nv_bfloat16*)y, n);
  return check_launch("gelu_bf16_kernel");
}
extern "C" int ftb_silu_f32_to_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n <= 0) return FTB_OK;
  silu_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(x, (__nv_bfloat16*)y, n);
  return check_launch("silu_kernel");
}
extern "C" int ftb_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream) {
  if (n <= 0) return FTB_OK;
  cast_f2b_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(x, (__nv_bfloat16*)y, n);
  return check_launch("cast_f2b_kernel");
}
extern "C" int ftb_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream) {
  if (n <= 0) return FTB_OK;
  cast_b2f_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>((const __nv_bfloat16*)x, y, n);
  return check_launch("cast_b2f_kernel");
}
extern "C" int ftb_fill_normal_bf16(void* out, int64_t n, uint64_t seed, float scale, void* stream) {
  if (n <= 0) return FTB_OK;
  fill_normal_bf16_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>((__nv_bfloat16*)out, n, seed, scale);
  return check_launch("fill_normal_bf16_kernel");
}
extern "C" int ftb_fill_normal_f32(float* out, int64_t n, uint64_t seed, float scale, void* stream) {
  if (n <= 0) return FTB_OK;
  fill_normal_f32_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(out, n, seed, scale);
  return check_launch("fill_normal_f32_kernel");
}
extern "C" int ftb_count_nonfinite(const float* x, int64_t n, int32_t* out, void* stream) {
  if (!out) return set_error(FTB_EINVAL, "count_nonfinite: null out");
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int32_t), S(stream));
  if (e != cudaSuccess) return set_cuda_error(e, "count_nonfinite memset");
  if (n <= 0) return FTB_OK;
  count_nonfinite_kernel<<<grid_for(n, 256), 256, 0, S(stream)>>>(x, n, out);
  return check_launch("count_nonfinite_kernel");
}

extern "C" int ftb_add_bcast_f32(const float* a, int64_t F, int64_t n, const float* b, int64_t Lb, float* out,
                                 void* stream) {
  if (!a || !b || !out || F <= 0 || n <= 0 || Lb <= 0) return set_error(FTB_EINVAL, "add_bcast: bad arguments");
  long long total = (long long)Lb * F * n;
  add_bcast_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>(a, b, out, F, n, total);
  return check_launch("add_bcast_kernel");
}

// ---------------------------------------------------------------- folded cross-attention
// The cross-attention keys/values (C·Wk, C·Wv of the L_c·A+1 conditioning tokens) are fixed
// for a chunk, so the projections fold through them (exact algebra, per layer and chunk):
//   S_h = (U·Wq_h)·K_h^T·s = U·(s·Wq_h·K_h^T)        At[(h,j)][k] = s·Σ_d K[j][h,d]·Wq^T[(h,d)][k]
//   out = Σ_h P_h·(V_h·Wo_h) = P·Bt^T                  Bt[n][(h,j)] = Σ_d Wo^T[n][(h,d)]·V[j][h,d]
// turning the two m×m projections per token into two m×(H·J) GEMMs (J = roundup(n_cond, 8)).
// At and Bt are two tensor-core GEMMs over the block-diagonal operands built here.
namespace ftb {

// Block-diagonal operands of the tensor-core fold: kbd[(h,j)][h*hd + d] = scale * K[j][h*hd + d],
// vbd[(h,j)][h*hd + d] = V[j][h*hd + d] for j < n_cond (kv = [n_cond][K | V]). Only the diagonal
// blocks are written; the caller keeps the rest (and rows j >= n_cond) zero.
__global__ void xattn_blockdiag_kernel(const __nv_bfloat16* __restrict__ kv, long long ldkv, int n_cond, int heads,
                                       int hd, int J, float scale, __nv_bfloat16* __restrict__ kbd,
                                       __nv_bfloat16* __restrict__ vbd, long long ld, int k_tile_segs) {
  const int m = heads * hd, v8 = hd / 8;
  const long long total = (long long)heads * n_cond * v8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int d8 = (int)(i % v8);
    const long long hj = i / v8;
    const int j = (int)(hj % n_cond), h = (int)(hj / n_cond);
    const int col = h * hd + d8 * 8;
    const uint4 kq = *reinterpret_cast<const uint4*>(kv + (long long)j * ldkv + col);
    const uint4 vq = *reinterpret_cast<const uint4*>(kv + (long long)j * ldkv + m + col);
    const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kq);
    uint4 ks;
    uint32_t* ko = reinterpret_cast<uint32_t*>(&ks);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(k2[e]);
      ko[e] = pack_bf16(f.x * scale, f.y * scale);
    }
    const long long row = (long long)h * J + j;
    // kbd rows optionally in the SEG_SOFTMAX tile order (k_tile_segs heads per 256-row tile)
    const long long krow = k_tile_segs > 0 ? (long long)(h / k_tile_segs) * 256 + (h % k_tile_segs) * J + j : row;
    *reinterpret_cast<uint4*>(kbd + krow * ld + col) = ks;
    *reinterpret_cast<uint4*>(vbd + row * ld + col) = vq;
  }
}

}  // namespace ftb

extern "C" int ftb_xattn_blockdiag(const void* kv, int64_t ldkv, int32_t n_cond, int32_t heads, int32_t head_dim,
                                   int32_t J, float scale, void* kbd, void* vbd, int64_t ld, int32_t k_tile_segs,
                                   void* stream) {
  if (!kv || !kbd || !vbd || n_cond <= 0 || J < n_cond || heads <= 0 || head_dim <= 0 || (head_dim % 8) ||
      (ldkv % 8) || (ld % 8) || ld < (int64_t)heads * head_dim || k_tile_segs < 0 || k_tile_segs * J > 256)
    return set_error(FTB_EINVAL, "xattn_blockdiag: bad arguments (n_cond <= J, head_dim / ldkv / ld % 8 == 0, "
                                 "k_tile_segs * J <= 256)");
  const long long total = (long long)heads * n_cond * (head_dim / 8);
  xattn_blockdiag_kernel<<<grid_for(total, 256), 256, 0, S(stream)>>>((const __nv_bfloat16*)kv, ldkv, n_cond, heads,
                                                                     head_dim, J, scale, (__nv_bfloat16*)kbd,
                                                                     (__nv_bfloat16*)vbd, ld, k_tile_segs);
  return check_launch("xattn_blockdiag_kernel");
}
