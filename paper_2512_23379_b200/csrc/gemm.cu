// Persistent warp-specialised tcgen05 GEMM with fused epilogues.
//
//   C[M,N] = A[M,K] . B[N,K]^T     bf16 x bf16 -> fp32 (TMEM) -> epilogue
//
// Roles (256 threads, 1 CTA / SM):
//   warp 0     TMA producer (one elected lane): A/B k-blocks -> smem ring
//   warp 1     MMA issuer (one lane): tcgen05.mma M=128 x N=BN x K=16, accumulators
//              double-buffered in TMEM so tile i+1's MMAs overlap tile i's epilogue
//   warp 2     TMEM allocator
//   warps 4-7  epilogue: tcgen05.ld -> bias / GELU / gate*residual / row-add / RoPE -> global
//
// Operand tiles are 128B-swizzled K-major (TMA SWIZZLE_128B box {64, rows});
// descriptors use SBO = 1024 B (8 rows x 128 B), K advance +32 B per UMMA_K.
// Replaces the reference's dense_forward (backends/reference.py:17-18) and the
// adds/activations that follow it in net.py:230-274.
#include <algorithm>

#include "common.cuh"
#include "ftb_internal.h"

namespace ftb {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;  // 4 control warps + 4 epilogue warps (EPG=2: + a second epilogue warpgroup)

struct GemmParams {
  int M, N, K;
  int kc;  // K per A chunk (K when a_chunks == 1)
  int kind;
  int rows_per_group;
  long long row_offset;
  const float* bias;
  const float* group_vec;
  long long group_ld;
  void* out;
  long long ldc;
  int heads, head_dim, hpr;
  ftb_rope3d rope;
  int has_rope;
  int group_m;                  // pair kernel: m-blocks per raster group (B reuse in L2)
  int n_peers;                  // > 0: QKV_ROPE / F32 stores go to peer-mapped buffers
  void* peers[FTB_MAX_PEERS];
  int staged;                   // pair kernel: residual epilogue through the per-warp smem tile
  int prefetch;                 // staged residual epilogue: L2 prefetch of the tile's h rows
  int tail_split;               // pair kernel, staged RESID: the partial last wave's tiles run as
                                // tail_split K-slices on separate pairs (1 = off)
  unsigned* tail_flags;         // per (tail tile, epilogue warp) slice counters, zero between launches
  int band_side, band_rows, band_tile, band_per_tile, band_k;  // block-diagonal operand (ftb_epilogue)
};

// K-block range of one pair tile: all of K, or (block-diagonal operand) the union of the bands
// of the tile's rows on the banded side; products outside it are exact zeros.
__device__ __forceinline__ void band_krange(const GemmParams& p, int m_blk, int n_blk, int num_kb, int& kb0, int& kb1) {
  kb0 = 0;
  kb1 = num_kb;
  if (p.band_k <= 0) return;
  const int r0 = (p.band_side ? n_blk : m_blk) * 256;
  const int r1 = min(r0 + 256, p.band_side ? p.N : p.M) - 1;
  auto band = [&](int r) {
    return p.band_tile > 0 ? (r / p.band_tile) * p.band_per_tile + (r % p.band_tile) / p.band_rows : r / p.band_rows;
  };
  const long long k0 = (long long)band(r0) * p.band_k, k1 = (long long)(band(r1) + 1) * p.band_k;
  const int a = (int)(k0 / GEMM_BK), b = (int)min((long long)num_kb, (k1 + GEMM_BK - 1) / GEMM_BK);
  if (a < b) {
    kb0 = a;
    kb1 = b;
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = GEMM_BM * GEMM_BK * 2;
  static constexpr int B_BYTES = BN * GEMM_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

// QKV_ROPE destination block [M][3][hpr][hd] for head group `dest`: a slice of `out`, or
// (Ulysses over peer memory) the peer-mapped receive block of rank `dest`.
__device__ __forceinline__ __nv_bfloat16* qkv_dest_block(const GemmParams& p, __nv_bfloat16* base, int dest) {
  if (p.n_peers) return reinterpret_cast<__nv_bfloat16*>(p.peers[dest]);
  return base + (long long)dest * p.M * 3 * ((long long)p.hpr * p.head_dim);
}



// RESID_F32 epilogue over a whole tile row (fast path: full 32-column chunks, aligned
// rows): the residual row segment of chunk c+1 is loaded while chunk c is finished, so two
// chunks of loads are in flight per thread (the plain path is latency-bound on these loads).
template <int WIDTH>
__device__ __forceinline__ bool resid_tile_pipelined(const GemmParams& p, uint32_t tmem_row, int gr, int gc_base) {
  if (p.kind != FTB_EPI_RESID_F32 || gc_base + WIDTH > p.N || (p.ldc & 3) || (p.group_vec && (p.group_ld & 3)))
    return false;
  const bool live = gr < p.M;
  const long long g = (p.rows_per_group > 0) ? (gr + p.row_offset) / p.rows_per_group : 0;
  float* orow = reinterpret_cast<float*>(p.out) + (long long)gr * p.ldc + gc_base;
  float4 hb[2][8];
  auto load = [&](int c, float4 (&dst)[8]) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = live ? reinterpret_cast<const float4*>(orow + c * 32)[q] : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  load(0, hb[0]);
#pragma unroll
  for (int c = 0; c < WIDTH / 32; ++c) {
    if (c + 1 < WIDTH / 32) load(c + 1, hb[(c + 1) & 1]);
    uint32_t r[32];
    tmem_ld32(tmem_row + c * 32, r);
    tmem_ld_wait();
    if (!live) continue;
    const int gc0 = gc_base + c * 32;
    const float* gate = p.group_vec ? p.group_vec + g * p.group_ld + gc0 : nullptr;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 acc = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                               __uint_as_float(r[4 * q + 3]));
      if (p.bias) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + gc0) + q);
        acc.x += b.x;
        acc.y += b.y;
        acc.z += b.z;
        acc.w += b.w;
      }
      const float4 gg = gate ? __ldg(reinterpret_cast<const float4*>(gate) + q) : make_float4(1.f, 1.f, 1.f, 1.f);
      float4 h = hb[c & 1][q];
      h.x += gg.x * acc.x;
      h.y += gg.y * acc.y;
      h.z += gg.z * acc.z;
      h.w += gg.w * acc.w;
      reinterpret_cast<float4*>(orow + c * 32)[q] = h;
    }
  }
  return true;
}

// Staged fp32 epilogue of the pair kernel (RESID_F32: h += gate * (acc + bias); F32:
// out = acc + bias; N % 32 == 0, 16-byte aligned rows). tcgen05.ld hands each thread one row;
// the thread parks a chunk's 32 accumulators in the warp's 4 KB smem tile (16-byte slots
// XOR-swizzled by row, conflict-free both ways) and the warp then walks its 32 rows
// row-contiguously: lane = (row % 4, float4 column), so every global float4 access covers
// four full 128-byte lines (the row-per-thread path touches 32 lines per instruction and is
// L1-wavefront bound at short K). For RESID, h of chunk c+1 is loaded before chunk c is
// combined. Same arithmetic as epilogue_chunk.
template <int WIDTH, bool GPF>
__device__ __forceinline__ void staged_tile_f32(const GemmParams& p, uint32_t tmem_row, int gr0, int gc_base,
                                                float4* stg, bool add_bias = true) {
  const int lane = lane_id();
  const int sub = lane >> 3, j = lane & 7;
  const bool resid = p.kind == FTB_EPI_RESID_F32;
  const int nch = min(WIDTH, p.N - gc_base) >> 5;  // chunks of 32 columns in this tile
  if (nch <= 0) return;                              // warp-uniform (column half past N)
  float* out = reinterpret_cast<float*>(p.out) + (long long)(gr0 + sub) * p.ldc + gc_base + 4 * j;
  const long long step = 4 * p.ldc;
  const int rows_left = p.M - gr0 - sub;  // row 4i+sub is live while 4i < rows_left
  const bool use_bias = add_bias && p.bias;
  const bool gated = resid && p.group_vec;
  // GPF (short K, where the epilogue bounds the tile): the warp's 32 rows almost always lie in one
  // gate group (a frame: 1170 rows); then the gate row is one float4 per chunk per thread, fetched
  // with the h rows of that chunk instead of inside the combine, where its latency sat on the
  // critical path (K = 1600: 206 -> 180 us); a block straddling two groups takes the per-row path.
  // Long K keeps the per-row loads: the extra registers spill there (+1-2 %).
  long long g0 = 0;
  bool uni = GPF;
  if (GPF && gated && p.rows_per_group > 0) {
    g0 = (gr0 + p.row_offset) / p.rows_per_group;
    uni = (min(gr0 + 31, p.M - 1) + p.row_offset) / p.rows_per_group == g0;
  }
  float4 hb[2][8], gb[2], bb[2];
  auto load = [&](int c, int s) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      hb[s][i] = (resid && 4 * i < rows_left) ? *reinterpret_cast<const float4*>(out + i * step + c * 32)
                                              : make_float4(0.f, 0.f, 0.f, 0.f);
    const int gc = gc_base + c * 32 + 4 * j;
    if (GPF) {
      gb[s] = (gated && uni) ? __ldg(reinterpret_cast<const float4*>(p.group_vec + g0 * p.group_ld + gc))
                             : make_float4(1.f, 1.f, 1.f, 1.f);
      bb[s] = use_bias ? __ldg(reinterpret_cast<const float4*>(p.bias + gc)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  load(0, 0);
#pragma unroll
  for (int c = 0; c < WIDTH / 32; ++c) {
    if (c >= nch) break;  // warp-uniform
    if (c + 1 < nch) load(c + 1, (c + 1) & 1);
    uint32_t r[32];
    tmem_ld32(tmem_row + c * 32, r);
    tmem_ld_wait();
#pragma unroll
    for (int q = 0; q < 8; ++q)
      stg[lane * 8 + (q ^ (lane & 7))] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
    __syncwarp();
    const int gc = gc_base + c * 32 + 4 * j;
    const float4 b = GPF ? bb[c & 1]
                         : (use_bias ? __ldg(reinterpret_cast<const float4*>(p.bias + gc)) : make_float4(0.f, 0.f, 0.f, 0.f));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = 4 * i + sub, row = gr0 + rr;
      float4 a = stg[rr * 8 + (j ^ (rr & 7))];
      if (4 * i < rows_left) {
        if (use_bias) {
          a.x += b.x;
          a.y += b.y;
          a.z += b.z;
          a.w += b.w;
        }
        float4* dst = reinterpret_cast<float4*>(out + i * step + c * 32);
        if (resid) {
          float4 gg = GPF ? gb[c & 1] : make_float4(1.f, 1.f, 1.f, 1.f);
          if (gated && !uni) {
            const long long g = (p.rows_per_group > 0) ? (row + p.row_offset) / p.rows_per_group : 0;
            gg = __ldg(reinterpret_cast<const float4*>(p.group_vec + g * p.group_ld + gc));
          }
          float4 h = hb[c & 1][i];
          h.x += gg.x * a.x;
          h.y += gg.y * a.y;
          h.z += gg.z * a.z;
          h.w += gg.w * a.w;
          *dst = h;
        } else {
          *dst = a;
        }
      }
    }
    __syncwarp();
  }
}

// FTB_EPI_SEG_SOFTMAX (folded cross-attention logits): a 256-column tile holds 256 / J whole
// J-column segments (one head's keys each; the rest of the tile is padding); the thread owns
// one row and turns each segment into softmax probabilities over its first n_cond columns
// (padded columns -> 0), written bf16 at column seg * J of `out`. Same arithmetic as
// xattn_softmax_kernel (elementwise.cu), so the fused and two-pass results agree bit for bit.
template <int J>
__device__ __forceinline__ void segsoftmax_tile(const GemmParams& p, uint32_t tmem_row, int gr, int n_blk, int part,
                                                int parts) {
  constexpr int SPT = 256 / J;
  const int n_cond = p.hpr;
  const int per = (SPT + parts - 1) / parts;
#pragma unroll 1
  for (int s = part * per; s < min(SPT, (part + 1) * per); ++s) {
    const int seg = n_blk * SPT + s;
    if (seg >= p.heads) break;  // warp-uniform
    uint32_t r[J];
#pragma unroll
    for (int k = 0; k < J / 8; ++k) tmem_ld8(tmem_row + s * J + 8 * k, *reinterpret_cast<uint32_t(*)[8]>(r + 8 * k));
    tmem_ld_wait();
    if (gr >= p.M) continue;
    float v[J];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      v[j] = __uint_as_float(r[j]);
      if (j < n_cond) mx = fmaxf(mx, v[j]);
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      v[j] = j < n_cond ? __expf(v[j] - mx) : 0.f;
      sum += v[j];
    }
    const float inv = 1.f / sum;
    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)gr * p.ldc + seg * J);
#pragma unroll
    for (int q = 0; q < J / 8; ++q)
      dst[q] = make_uint4(pack_bf16(v[8 * q] * inv, v[8 * q + 1] * inv), pack_bf16(v[8 * q + 2] * inv, v[8 * q + 3] * inv),
                          pack_bf16(v[8 * q + 4] * inv, v[8 * q + 5] * inv), pack_bf16(v[8 * q + 6] * inv, v[8 * q + 7] * inv));
  }
}

// part / parts: this epilogue warpgroup's share of the tile's segments
__device__ __forceinline__ void segsoftmax_dispatch(const GemmParams& p, uint32_t tmem_row, int gr, int n_blk,
                                                    int part = 0, int parts = 1) {
  switch (p.head_dim) {  // J
    case 8: segsoftmax_tile<8>(p, tmem_row, gr, n_blk, part, parts); break;
    case 16: segsoftmax_tile<16>(p, tmem_row, gr, n_blk, part, parts); break;
    case 24: segsoftmax_tile<24>(p, tmem_row, gr, n_blk, part, parts); break;
    case 32: segsoftmax_tile<32>(p, tmem_row, gr, n_blk, part, parts); break;
    case 40: segsoftmax_tile<40>(p, tmem_row, gr, n_blk, part, parts); break;
    default: segsoftmax_tile<48>(p, tmem_row, gr, n_blk, part, parts); break;
  }
}

// Epilogue for one thread: row `gr`, 32 fp32 accumulators for columns [gc0, gc0+32).
// Every loop over the 32 accumulators is fully unrolled with per-element predicates (no
// data-dependent trip counts), so v[] stays in registers: a dynamic index anywhere in this
// function puts the whole array in local memory (seen as STL/LDL on the short-K 1.3B GEMMs).
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int gr, int gc0, float (&v)[32]) {
  const int N = p.N;
  const bool full = (gc0 + 32 <= N);
  if (p.bias) {
    if (full && !(reinterpret_cast<uintptr_t>(p.bias + gc0) & 15)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 b = __ldg(reinterpret_cast<const float4*>(p.bias + gc0) + q);
        v[4 * q] += b.x;
        v[4 * q + 1] += b.y;
        v[4 * q + 2] += b.z;
        v[4 * q + 3] += b.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (gc0 + j < N) v[j] += __ldg(p.bias + gc0 + j);
    }
  }
  const long long g = (p.rows_per_group > 0) ? (gr + p.row_offset) / p.rows_per_group : 0;
  switch (p.kind) {
    case FTB_EPI_GELU_BF16:
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_tanh(v[j]);
      // fallthrough
    case FTB_EPI_BF16: {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.out) + (long long)gr * p.ldc + gc0;
      if (full && ((p.ldc & 7) == 0)) {
        uint4* o4 = reinterpret_cast<uint4*>(o);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
          w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
          w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
          w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
          o4[q] = w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (gc0 + j < N) o[j] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    case FTB_EPI_F32: {
      if (p.n_peers) {  // replicated store: the all-gather of the result rides the epilogue
        for (int r = 0; r < p.n_peers; ++r) {
          float* o = reinterpret_cast<float*>(p.peers[r]) + (long long)gr * p.ldc + gc0;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (gc0 + j < N) o[j] = v[j];
        }
        break;
      }
      float* o = reinterpret_cast<float*>(p.out) + (long long)gr * p.ldc + gc0;
      if (full && ((p.ldc & 3) == 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (gc0 + j < N) o[j] = v[j];
      }
      break;
    }
    case FTB_EPI_RESID_F32: {
      float* o = reinterpret_cast<float*>(p.out) + (long long)gr * p.ldc + gc0;
      const float* gate = p.group_vec ? p.group_vec + g * p.group_ld + gc0 : nullptr;
      if (full && ((p.ldc & 3) == 0) && (!gate || (p.group_ld & 3) == 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 r = reinterpret_cast<float4*>(o)[q];
          float4 gg = gate ? __ldg(reinterpret_cast<const float4*>(gate) + q) : make_float4(1.f, 1.f, 1.f, 1.f);
          r.x += gg.x * v[4 * q + 0];
          r.y += gg.y * v[4 * q + 1];
          r.z += gg.z * v[4 * q + 2];
          r.w += gg.w * v[4 * q + 3];
          reinterpret_cast<float4*>(o)[q] = r;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (gc0 + j < N) o[j] += (gate ? gate[j] : 1.f) * v[j];
      }
      break;
    }
    case FTB_EPI_ROWADD_F32: {
      float* o = reinterpret_cast<float*>(p.out) + (long long)gr * p.ldc + gc0;
      const float* add = p.group_vec ? p.group_vec + g * p.group_ld + gc0 : nullptr;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (gc0 + j < N) o[j] = v[j] + (add ? __ldg(add + j) : 0.f);
      break;
    }
    case FTB_EPI_QKV_ROPE: {
      const int m = p.heads * p.head_dim;
      const long long token = gr + p.row_offset;
      __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(p.out);
      if (full && (p.head_dim & 31) == 0) {
        // fast path: the 32 columns lie in one head -> one destination run of 64 bytes
        const int which = gc0 / m;
        const int cm = gc0 - which * m;
        const int h = cm / p.head_dim;
        const int d0 = cm - h * p.head_dim;
        if (which < 2 && p.has_rope) {
          const int half = p.head_dim >> 1;
          const float4* cs = reinterpret_cast<const float4*>(p.rope.cos_full + token * half + (d0 >> 1));
          const float4* sn = reinterpret_cast<const float4*>(p.rope.sin_full + token * half + (d0 >> 1));
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 c4 = __ldg(cs + q4), s4 = __ldg(sn + q4);
            const float cc[4] = {c4.x, c4.y, c4.z, c4.w}, ss[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int j = 8 * q4 + 2 * e;
              const float a = v[j] * cc[e] - v[j + 1] * ss[e];
              const float b = v[j] * ss[e] + v[j + 1] * cc[e];
              v[j] = a;
              v[j + 1] = b;
            }
          }
        }
        const int dest = h / p.hpr;
        const int hl = h - dest * p.hpr;
        uint4* o4 = reinterpret_cast<uint4*>(qkv_dest_block(p, base, dest) +
                                             ((long long)gr * 3 + which) * ((long long)p.hpr * p.head_dim) +
                                             (long long)hl * p.head_dim + d0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 w;
          w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
          w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
          w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
          w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
          o4[q] = w;
        }
        break;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const int c = gc0 + j;
        if (c < N) {
          const int which = c / m;
          const int cm = c - which * m;
          const int h = cm / p.head_dim;
          const int d = cm - h * p.head_dim;
          float x0 = v[j], x1 = v[j + 1];
          if (which < 2 && p.has_rope) {
            const long long ix = token * (p.head_dim >> 1) + (d >> 1);
            const float cr = __ldg(p.rope.cos_full + ix), sr = __ldg(p.rope.sin_full + ix);
            const float a = x0 * cr - x1 * sr;
            x1 = x0 * sr + x1 * cr;
            x0 = a;
          }
          const int dest = h / p.hpr;
          const int hl = h - dest * p.hpr;
          const long long idx =
              ((long long)gr * 3 + which) * ((long long)p.hpr * p.head_dim) + (long long)hl * p.head_dim + d;
          *reinterpret_cast<uint32_t*>(qkv_dest_block(p, base, dest) + idx) = pack_bf16(x0, x1);
        }
      }
      break;
    }
    default:
      break;
  }
}

template <int BN, int EPG>
__global__ void __launch_bounds__(GEMM_THREADS + (EPG - 1) * 128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + C::STAGES;
  uint64_t* tfull_bar = empty_bar + C::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  const int num_m = (p.M + GEMM_BM - 1) / GEMM_BM;
  const int num_n = (p.N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (p.K + GEMM_BK - 1) / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);  // one arrive per epilogue warp
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
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], C::STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          const int chunk = k0 / p.kc;
          tma_load_3d(sa, &tmA, &full_bar[stage], k0 - chunk * p.kc, m_blk * GEMM_BM, chunk);
          tma_load_2d(sb, &tmB, &full_bar[stage], k0, n_blk * BN);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer: warp-converged, one elected lane issues (uniform descriptors)
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(GEMM_BM, BN, 0, 0);
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
          for (int k = 0; k < GEMM_BK / 16; ++k) {
            uint64_t ad = sdesc_sw128(sa + k * 32, 16, 1024);
            uint64_t bd = sdesc_sw128(sb + k * 32, 16, 1024);
            mma_bf16_ss_elect(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
          }
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
    // ---------------- epilogue (EPG=2: warpgroup eg drains accumulator eg, every other tile, so
    // a tile's epilogue has two mainloops of time — short-K GEMMs are epilogue-bound otherwise)
    const int q = warp & 3;  // TMEM lane quadrant
    const int eg = (warp - 4) >> 2;
    int it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      if (EPG == 2 && (it & 1) != eg) continue;
      const int m_blk = tile / num_n, n_blk = tile - (tile / num_n) * num_n;
      const int acc = it & 1;
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const int gr = m_blk * GEMM_BM + q * 32 + lane;
      if (BN == 256 && p.kind == FTB_EPI_SEG_SOFTMAX)
        segsoftmax_dispatch(p, tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, gr, n_blk);
      else if (!resid_tile_pipelined<BN>(p, tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN, gr, n_blk * BN))
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        const int gc0 = n_blk * BN + c0;
        if (gc0 >= p.N) break;  // warp-uniform
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c0, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (gr < p.M) epilogue_chunk(p, gr, gc0, v);
      }
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

// ------------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): one 256 x 256 tile per pair, UMMA M=256, each CTA
// stages its 128 rows of A and 128 rows of B^T (half the operand bytes of two 1-CTA
// tiles), 6-stage ring, TMEM accumulators double-buffered (2 x 256 columns). Tiles
// are rasterised in groups of GROUP_M m-blocks so a wave of pairs shares B in L2.
constexpr int PAIR_STAGES = 6;
constexpr int PAIR_A_BYTES = 128 * GEMM_BK * 2;
constexpr int PAIR_B_BYTES = 128 * GEMM_BK * 2;
constexpr int PAIR_STAGE_BYTES = PAIR_A_BYTES + PAIR_B_BYTES;
constexpr int PAIR_EPI_STAGE = 8 * 4096;  // per-epilogue-warp 32 x 32 fp32 staging tiles
constexpr int PAIR_SMEM = PAIR_STAGES * PAIR_STAGE_BYTES + 1024 + 256 + PAIR_EPI_STAGE;
// HT variant (short-K fp32 residual GEMMs): a 5-stage ring and, per epilogue warp, two of the
// four 32 x 32 fp32 boxes (128-byte swizzled) of its 32-row x 128-column h tile in shared memory;
// box c + 2 reuses box c's buffer once that box's TMA store has read it. Ring depth beats box
// count: 5 stages / 2 boxes vs 4 / 3 at 10530 rows: N 5120 K 1600 158.6 vs 170.3 us, N 1536
// K 1536 70.4 vs 83.2, K 480 56.2 vs 60.0 (3 stages / 4 boxes lost 2-9 % at K >= 1024).
constexpr int PAIR_STAGES_HT = 5;
constexpr int PAIR_BOXES_HT = 2;
constexpr int PAIR_SMEM_HT = PAIR_STAGES_HT * PAIR_STAGE_BYTES + 1024 + 1024 + 8 * PAIR_BOXES_HT * 4096;

__device__ __forceinline__ void pair_raster(int tile, int num_m, int num_n, int group_m, int& m_blk, int& n_blk) {
  const int group = group_m * num_n;
  const int g = tile / group;
  const int first_m = g * group_m;
  const int gm = min(num_m - first_m, group_m);
  const int local = tile - g * group;
  m_blk = first_m + local % gm;
  n_blk = local / gm;
}

// Work items of the pair kernel. With tail_split = s > 1 the R = num_tiles % n_clusters tiles
// of the partial last wave run as s K-slices each on s different pairs (items F + s*t + part,
// F = num_tiles - R, all in the last round since s*R <= n_clusters). Slice `part` adds its
// partial product into h after slice part-1 has (per epilogue warp counter), and only slice 0
// adds the bias: h + g*(a0 + b) + g*a1 ..., fixed order, so the result is deterministic.
struct PairItem {
  int tile, kb0, kb1, part, slot;  // slot: tail tile index (-1 for a whole tile)
};
__device__ __forceinline__ PairItem pair_item(int i, int num_tiles, int n_clusters, int s, int num_kb) {
  const int R = s > 1 ? num_tiles % n_clusters : 0;
  const int F = num_tiles - R;
  if (i < F) return PairItem{i, 0, num_kb, 0, -1};
  const int t = (i - F) / s, part = (i - F) - t * s;
  return PairItem{F + t, part * num_kb / s, (part + 1) * num_kb / s, part, t};
}
__device__ __forceinline__ int pair_num_items(int num_tiles, int n_clusters, int s) {
  return s > 1 ? num_tiles + (s - 1) * (num_tiles % n_clusters) : num_tiles;
}

__device__ __forceinline__ void tail_wait(const unsigned* flag, unsigned want) {
  if (lane_id() == 0) {
    const long long t0 = clock64();
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      if (v >= want) break;
      __nanosleep(64);
      if (clock64() - t0 > (1LL << 33)) __trap();  // ~4 s: a lost slice would hang the box
    }
  }
  __syncwarp();
  __threadfence();
}

template <int EPG, bool STAGED, bool GPF = false, bool HT = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS + (EPG - 1) * 128, 1)
    gemm_tc_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmH, const GemmParams p) {
  constexpr int NSTG = HT ? PAIR_STAGES_HT : PAIR_STAGES;
  constexpr int HB = HT ? PAIR_BOXES_HT : 1;   // h boxes per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + NSTG * PAIR_STAGE_BYTES);
  uint64_t* empty_bar = full_bar + NSTG;
  uint64_t* tfull_bar = empty_bar + NSTG;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int num_m = (p.M + 255) / 256;
  const int num_n = (p.N + 255) / 256;
  const int num_tiles = num_m * num_n;
  const int num_kb = (p.K + GEMM_BK - 1) / GEMM_BK;
  const int num_items = pair_num_items(num_tiles, n_clusters, p.tail_split);

  uint64_t* h_bar = reinterpret_cast<uint64_t*>(smem + NSTG * PAIR_STAGE_BYTES + 512);  // HT: [8 warps][4 boxes]
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (HT) {
      tma_prefetch(&tmH);
      for (int i = 0; i < 32; ++i) mbar_init(&h_bar[i], 1);
    }
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      // epilogue warps x 2 CTAs arrive (leader's copy is the one used): 4 per CTA, or all 8 when
      // both warpgroups drain every tile (EPG=2 column split)
      mbar_init(&tempty_bar[s], EPG == 2 ? 16 : 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int item = cluster; item < num_items; item += n_clusters) {
        PairItem w = pair_item(item, num_tiles, n_clusters, p.tail_split, num_kb);
        int m_blk, n_blk;
        pair_raster(w.tile, num_m, num_n, p.group_m, m_blk, n_blk);
        if (p.band_k > 0) band_krange(p, m_blk, n_blk, num_kb, w.kb0, w.kb1);  // host: no tail split then
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * PAIR_STAGE_BYTES;
          uint8_t* sb = sa + PAIR_A_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], 2 * PAIR_STAGE_BYTES);
          const int k0 = kb * GEMM_BK;
          const int chunk = k0 / p.kc;
          tma_load_3d_pair(sa, &tmA, &full_bar[stage], k0 - chunk * p.kc, m_blk * 256 + rank * 128, chunk);
          tma_load_2d_pair(sb, &tmB, &full_bar[stage], k0, n_blk * 256 + rank * 128);
          if (++stage == NSTG) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // warp-converged issue on the leader CTA, one elected lane
      __syncwarp();
      constexpr uint32_t idesc = idesc_bf16(256, 256, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = cluster; item < num_items; item += n_clusters, ++it) {
        PairItem w = pair_item(item, num_tiles, n_clusters, p.tail_split, num_kb);
        if (p.band_k > 0) {
          int m_blk, n_blk;
          pair_raster(w.tile, num_m, num_n, p.group_m, m_blk, n_blk);
          band_krange(p, m_blk, n_blk, num_kb, w.kb0, w.kb1);
        }
        const int acc = it & 1;
        mbar_wait(&tempty_bar[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * 256;
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * PAIR_STAGE_BYTES);
          const uint32_t sb = sa + PAIR_A_BYTES;
#pragma unroll
          for (int k = 0; k < GEMM_BK / 16; ++k)
            mma_bf16_ss_pair_elect(tmem_d, sdesc_sw128(sa + k * 32, 16, 1024), sdesc_sw128(sb + k * 32, 16, 1024), idesc,
                             (kb != w.kb0 || k) ? 1u : 0u);
          mma_commit_pair_elect(&empty_bar[stage], 0x3);
          if (++stage == NSTG) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit_pair_elect(&tfull_bar[acc], 0x3);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int eg = (warp - 4) >> 2;  // epilogue warpgroup
    // EPG=2 column split: each warpgroup drains 128 of every tile's 256 columns, so a tile's
    // epilogue takes half as long (with two TMEM accumulators an epilogue must finish within
    // one mainloop whichever warpgroup runs it); otherwise warpgroup eg drains accumulator eg
    constexpr bool split = EPG == 2;
    const int col0 = split ? eg * 128 : 0;
    uint32_t h_phase = 0;  // HT: parity bit per h box barrier (edge tiles may use fewer boxes)
    int it = 0;
    for (int item = cluster; item < num_items; item += n_clusters, ++it) {
      if (EPG == 2 && !split && (it & 1) != eg) continue;
      const PairItem w = pair_item(item, num_tiles, n_clusters, p.tail_split, num_kb);
      int m_blk, n_blk;
      pair_raster(w.tile, num_m, num_n, p.group_m, m_blk, n_blk);
      const int acc = it & 1;
      const int gr = m_blk * 256 + rank * 128 + q * 32 + lane;
      const int width = split ? 128 : 256;
      const int gcb = n_blk * 256 + col0;
      // HT: this warp's h tile (rows gr - lane .. +32, columns gcb .. +128) is fetched by TMA
      // before the accumulator is even ready; the boxes of the previous tile must have left
      // shared memory first (their TMA stores read it)
      float4* hbuf = reinterpret_cast<float4*>(smem + NSTG * PAIR_STAGE_BYTES + 1024 + (warp - 4) * HB * 4096);
      const int hch = HT ? max(0, min(width, p.N - gcb) >> 5) : 0;
      if (HT && lane == 0) {
        bulk_wait_read0();
        for (int c = 0; c < hch && c < HB; ++c) {
          mbar_arrive_expect_tx(&h_bar[(warp - 4) * 4 + c], 4096);
          tma_load_2d(hbuf + c * 256, &tmH, &h_bar[(warp - 4) * 4 + c], gcb + 32 * c, gr - lane);
        }
      }
      if (!HT && STAGED && p.prefetch && p.kind == FTB_EPI_RESID_F32 && gr < p.M && gcb < p.N) {
        // pull this thread's row segment of h (<= 1 KB) into L2 while the tile's MMAs run, so
        // the epilogue's h loads hit L2 (DRAM latency x the few loads in flight per warp otherwise bound it)
        const float* hrow = reinterpret_cast<const float*>(p.out) + (long long)gr * p.ldc + gcb;
        const uint32_t bytes = (uint32_t)min(width, p.N - gcb) * 4;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(hrow), "r"(bytes) : "memory");
      }
      mbar_wait(&tfull_bar[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t trow = tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256 + col0;
      if constexpr (HT) {  // host: RESID_F32, EPG 2, N % 32 == 0, no tail split
        // thread = row (TMEM lane): its 32-column slice of the swizzled h box, h += g*(acc + bias)
        // in place, then one TMA store per box (rows past M / columns past N are clipped)
        const float4* gv = nullptr;
        if (p.group_vec) {
          const long long g = p.rows_per_group > 0 ? (min(gr, p.M - 1) + p.row_offset) / p.rows_per_group : 0;
          gv = reinterpret_cast<const float4*>(p.group_vec + g * p.group_ld + gcb);
        }
        const float4* bv = p.bias ? reinterpret_cast<const float4*>(p.bias + gcb) : nullptr;
        for (int c = 0; c < hch; ++c) {
          const int b = c % HB;
          uint32_t r[32];
          tmem_ld32(trow + c * 32, r);
          mbar_wait(&h_bar[(warp - 4) * 4 + b], (h_phase >> b) & 1u);
          h_phase ^= 1u << b;
          tmem_ld_wait();
          float4* row = hbuf + b * 256 + lane * 8;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float4 a = make_float4(__uint_as_float(r[4 * k]), __uint_as_float(r[4 * k + 1]), __uint_as_float(r[4 * k + 2]),
                                   __uint_as_float(r[4 * k + 3]));
            if (bv) {
              const float4 b = __ldg(bv + c * 8 + k);
              a.x += b.x;
              a.y += b.y;
              a.z += b.z;
              a.w += b.w;
            }
            const float4 gg = gv ? __ldg(gv + c * 8 + k) : make_float4(1.f, 1.f, 1.f, 1.f);
            float4 h = row[k ^ (lane & 7)];
            h.x = fmaf(gg.x, a.x, h.x);
            h.y = fmaf(gg.y, a.y, h.y);
            h.z = fmaf(gg.z, a.z, h.z);
            h.w = fmaf(gg.w, a.w, h.w);
            row[k ^ (lane & 7)] = h;
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmH, hbuf + b * 256, gcb + 32 * c, gr - lane);
            bulk_commit();
            if (c + HB < hch) {  // box b takes chunk c + HB once its store has read it
              bulk_wait_read0();
              mbar_arrive_expect_tx(&h_bar[(warp - 4) * 4 + b], 4096);
              tma_load_2d(hbuf + b * 256, &tmH, &h_bar[(warp - 4) * 4 + b], gcb + 32 * (c + HB), gr - lane);
            }
          }
        }
      } else if (STAGED) {  // host guarantees RESID_F32 / F32 (no peers), N % 32 == 0, aligned rows / gate / bias
        float4* stg = reinterpret_cast<float4*>(smem + NSTG * PAIR_STAGE_BYTES + 256 + (warp - 4) * 4096);
        // K-slice of a tail tile: this warp's rows/columns of slice part-1 must be in h first
        if (w.slot >= 0 && w.part > 0)
          tail_wait(p.tail_flags + w.slot * 16 + rank * 8 + eg * 4 + q, (unsigned)w.part);
        staged_tile_f32<split ? 128 : 256, GPF>(p, trow, gr - lane, gcb, stg, w.part == 0);
        const PairItem w2 = pair_item(item, num_tiles, n_clusters, p.tail_split, num_kb);  // cheaper than live regs
        if (w2.slot >= 0) {
          __threadfence();
          __syncwarp();
          // the last slice is the only reader left: it re-arms the counter for the next launch
          unsigned* flag = p.tail_flags + w2.slot * 16 + rank * 8 + eg * 4 + q;
          if (lane == 0) {
            if (w2.part + 1 < p.tail_split) atomicAdd(flag, 1u);
            else atomicExch(flag, 0u);
          }
        }
      } else if (p.kind == FTB_EPI_SEG_SOFTMAX) {
        segsoftmax_dispatch(p, tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256, gr, n_blk, split ? eg : 0,
                            split ? 2 : 1);
      } else if (!resid_tile_pipelined<split ? 128 : 256>(p, trow, gr, gcb))
#pragma unroll 1
      for (int c0 = col0; c0 < col0 + width; c0 += 32) {
        const int gc0 = n_blk * 256 + c0;
        if (gc0 >= p.N) break;
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * 256 + c0, r);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (gr < p.M) epilogue_chunk(p, gr, gc0, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tempty_bar[acc], 0);
    }
  }
  if (HT && warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<512>(tmem_base);
}

template <int EPG, bool STAGED, bool GPF = false, bool HT = false>
static int launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t stream,
                            const CUtensorMap* th = nullptr) {
  constexpr int SMEM = HT ? PAIR_SMEM_HT : PAIR_SMEM;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_pair_kernel<EPG, STAGED, GPF, HT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm pair smem attribute");
    configured = true;
  }
  const int tiles = ((p.M + 255) / 256) * ((p.N + 255) / 256);
  const int max_pairs = sm_count() / 2;
  const int pairs = tiles < max_pairs ? tiles : max_pairs;
  gemm_tc_pair_kernel<EPG, STAGED, GPF, HT><<<2 * pairs, GEMM_THREADS + (EPG - 1) * 128, SMEM, stream>>>(
      ta, tb, th ? *th : tb, p);
  return check_launch("gemm_tc_pair_kernel");
}

template <int BN, int EPG>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<BN, EPG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "gemm smem attribute");
    configured = true;
  }
  const int tiles = ((p.M + GEMM_BM - 1) / GEMM_BM) * ((p.N + BN - 1) / BN);
  const int grid = tiles < sm_count() ? tiles : sm_count();
  gemm_tc_kernel<BN, EPG><<<grid, GEMM_THREADS + (EPG - 1) * 128, C::SMEM, stream>>>(ta, tb, p);
  return check_launch("gemm_tc_kernel");
}

}  // namespace ftb

using namespace ftb;

// Split-K tail counters: FTB_TAIL_COUNTER_WORDS = FTB_TAIL_SLOTS x 16 words per caller buffer.
constexpr int FTB_TAIL_SLOTS = FTB_TAIL_COUNTER_WORDS / 16;  // >= n_clusters (74 on B200)

extern "C" int ftb_gemm_bf16(const void* A, int64_t lda, int32_t a_chunks, int64_t a_chunk_stride, const void* B,
                             int64_t ldb, int32_t M, int32_t N, int32_t K, const ftb_epilogue* epi, void* stream) {
  if (!A || !B || !epi || !epi->out) return set_error(FTB_EINVAL, "gemm: null pointer");
  if (M <= 0 || N <= 0 || K <= 0) return set_error(FTB_EINVAL, "gemm: empty problem");
  if ((lda & 7) || (ldb & 7)) return set_error(FTB_EINVAL, "gemm: lda/ldb must be multiples of 8 elements");
  if (a_chunks < 1) a_chunks = 1;
  if (K % a_chunks) return set_error(FTB_EINVAL, "gemm: K not divisible by a_chunks");
  const int kc = K / a_chunks;
  if (a_chunks > 1 && (kc % GEMM_BK)) return set_error(FTB_EINVAL, "gemm: K/a_chunks must be a multiple of 64");
  if (a_chunks > 1 && (a_chunk_stride & 7)) return set_error(FTB_EINVAL, "gemm: chunk stride alignment");
  if (epi->kind < FTB_EPI_BF16 || epi->kind > FTB_EPI_SEG_SOFTMAX) return set_error(FTB_EINVAL, "gemm: bad epilogue");
  if (epi->kind == FTB_EPI_SEG_SOFTMAX) {
    const int J = epi->head_dim, segs = epi->heads, n_cond = epi->heads_per_rank;
    if (J < 8 || J > 48 || (J % 8) || segs <= 0 || n_cond <= 0 || n_cond > J || epi->bias || epi->n_peers ||
        (epi->ldc % 8) || epi->ldc < (int64_t)segs * J || N != (segs + 256 / J - 1) / (256 / J) * 256)
      return set_error(FTB_EINVAL, "gemm: SEG_SOFTMAX needs J % 8 == 0 <= 48, 0 < n_cond <= J, no bias/peers, "
                                   "N = 256 * ceil(segments / (256 / J)), ldc >= segments * J");
  }
  if (epi->kind == FTB_EPI_QKV_ROPE) {
    if (epi->heads <= 0 || epi->head_dim <= 0 || (epi->head_dim & 1) || epi->heads_per_rank <= 0 ||
        epi->heads % epi->heads_per_rank || N != 3 * epi->heads * epi->head_dim)
      return set_error(FTB_EINVAL, "gemm: bad QKV layout");
  }
  if (epi->n_peers < 0 || epi->n_peers > FTB_MAX_PEERS) return set_error(FTB_EINVAL, "gemm: bad peer count");
  if (epi->n_peers) {
    if (epi->kind != FTB_EPI_QKV_ROPE && epi->kind != FTB_EPI_F32)
      return set_error(FTB_EINVAL, "gemm: peer stores need the QKV_ROPE or F32 epilogue");
    if (epi->kind == FTB_EPI_QKV_ROPE && epi->n_peers != epi->heads / epi->heads_per_rank)
      return set_error(FTB_EINVAL, "gemm: QKV peers must equal heads / heads_per_rank");
    for (int i = 0; i < epi->n_peers; ++i)
      if (!epi->peer_out[i]) return set_error(FTB_EINVAL, "gemm: null peer pointer");
  }
  // kernel selection of this call (ftb_epilogue.variant; 0 = product defaults)
  const int variant = epi->variant;
  if (variant < 0 || (variant & 3) == 3 || variant > 63)
    return set_error(FTB_EINVAL, "gemm: variant must be 0/1/2 (auto / single CTA / CTA pair) + 4 (row-per-thread "
                                 "residual epilogue) + 8 (no h prefetch) + 16 (one epilogue warpgroup at long K) + 32 "
                                 "(no TMA-staged short-K residual epilogue)");
  if (epi->raster_group < 0) return set_error(FTB_EINVAL, "gemm: raster_group must be >= 0");
  GemmParams p{};
  p.n_peers = epi->n_peers;
  p.staged = (variant & 4) ? 0 : 1;
  // short K only: there the h rows must stream at DRAM rate behind a short mainloop; at long K
  // the prefetched rows just displace A/B panels from L2 (measured -3..-4 % at K >= 5120)
  p.prefetch = !(variant & 8) && K <= 2048;
  for (int i = 0; i < epi->n_peers; ++i) p.peers[i] = epi->peer_out[i];
  p.M = M;
  p.N = N;
  p.K = K;
  p.kc = kc;
  p.kind = epi->kind;
  p.rows_per_group = epi->rows_per_group;
  p.row_offset = epi->row_offset;
  p.bias = epi->bias;
  p.group_vec = epi->group_vec;
  p.group_ld = epi->group_ld;
  p.out = epi->out;
  p.ldc = epi->ldc;
  p.heads = epi->heads;
  p.head_dim = epi->head_dim;
  p.hpr = epi->heads_per_rank;
  p.has_rope = epi->rope != nullptr;
  if (epi->band_k > 0) {
    if (epi->band_rows <= 0 || epi->band_side < 0 || epi->band_side > 1 ||
        (epi->band_tile > 0 && (epi->band_per_tile <= 0 || epi->band_tile < epi->band_rows)) || a_chunks > 1)
      return set_error(FTB_EINVAL, "gemm: bad block-diagonal band description");
    p.band_side = epi->band_side;
    p.band_rows = epi->band_rows;
    p.band_tile = epi->band_tile;
    p.band_per_tile = epi->band_per_tile;
    p.band_k = epi->band_k;
  }
  if (epi->rope) p.rope = *epi->rope;

  const bool pair = (variant & 3) == 2 || ((variant & 3) == 0 && M >= 256 && N >= 256);
  int BN = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  // few m-blocks (cond-token K/V projections, M = 37): narrower tiles until the grid covers
  // the SMs, so the weight stream is spread over every SM's load path
  while (!pair && BN > 64 && epi->kind != FTB_EPI_SEG_SOFTMAX &&
         (long long)((M + GEMM_BM - 1) / GEMM_BM) * ((N + BN - 1) / BN) < sm_count())
    BN >>= 1;
  {
    // raster group: enough 256-row m-blocks that their A panels (~40 MB) stay in L2 while
    // the B panel streams past once per group
    const long long panel = 256LL * K * 2;
    int gmax = (int)(40LL * 1024 * 1024 / (panel > 0 ? panel : 1));
    if (epi->raster_group > 0) gmax = epi->raster_group;
    p.group_m = gmax < 8 ? 8 : gmax;
  }
  CUtensorMap ta, tb;
  // A: 3D {kc, M, chunks}
  {
    uint64_t dims[3] = {(uint64_t)kc, (uint64_t)M, (uint64_t)a_chunks};
    uint64_t strides[2] = {(uint64_t)lda * 2, (uint64_t)(a_chunks > 1 ? a_chunk_stride : (int64_t)lda * M) * 2};
    uint32_t box[3] = {GEMM_BK, GEMM_BM, 1};
    int rc = make_tmap_bf16(&ta, A, 3, dims, strides, box);
    if (rc) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)K, (uint64_t)N};
    uint64_t strides[1] = {(uint64_t)ldb * 2};
    uint32_t box[2] = {GEMM_BK, pair ? 128u : (uint32_t)BN};
    int rc = make_tmap_bf16(&tb, B, 2, dims, strides, box);
    if (rc) return rc;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // short K: the per-tile mainloop is shorter than one epilogue warpgroup's drain -> two groups
  // (+ residual GEMMs at any K: the column-split fp32 epilogue drains h in half the time; FFN2
  // K=13824 1232-1281 -> 1408 TFLOP/s, chunk GEMM time -4.5 ms; bf16 epilogues lose at long K)
  const bool epg2 = K <= 2048 || (!(variant & 16) && epi->kind == FTB_EPI_RESID_F32);
  if (pair) {
    auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool staged = p.staged && (p.kind == FTB_EPI_RESID_F32 || (p.kind == FTB_EPI_F32 && !p.n_peers)) &&
                        N % 32 == 0 && !(p.ldc & 3) && al16(p.out) &&
                        (!p.group_vec || (!(p.group_ld & 3) && al16(p.group_vec))) && (!p.bias || al16(p.bias));
    p.tail_split = 1;
    if (staged && epi->tail_counters && p.kind == FTB_EPI_RESID_F32 && p.band_k <= 0) {
      // partial last wave of R < n_clusters / 2 tiles: run them as K-slices on the idle pairs
      // (FFN2 / O-proj at M = 10530, N = 5120: 840 tiles = 11.35 waves of 74 pairs -> 11.5)
      const int tiles = ((M + 255) / 256) * ((N + 255) / 256);
      const int n_clusters = std::min(tiles, sm_count() / 2);
      const int R = tiles % n_clusters;
      const int num_kb = (K + GEMM_BK - 1) / GEMM_BK;
      // long K only: slice p's epilogue waits for slice p-1's, so the tail costs K/s of mainloop
      // plus s epilogues; measured (scripts/gemm_tail_ab.py, interleaved medians) FFN2 K = 13824
      // -3.7 %, K = 8960 -2.7 %, but K = 5120 +7 % and K <= 1600 +8..15 % (epilogue-heavy)
      int sp = (R && num_kb >= 128) ? std::min(4, n_clusters / R) : 1;
      while (sp > 1 && num_kb / sp < 8) --sp;
      if (sp > 1 && n_clusters <= FTB_TAIL_SLOTS) {
        p.tail_flags = epi->tail_counters;
        p.tail_split = sp;
      }
    }
    if (staged && K <= 2048 && epg2 && p.kind == FTB_EPI_RESID_F32 && p.tail_split <= 1 && !(variant & 32)) {
      // short-K fp32 residual GEMMs: h tiles in and out by TMA (the per-thread h loads of the
      // staged epilogue bound these shapes at ~2 TB/s of h traffic). Measured vs the staged
      // epilogue (10530 rows): N 1536 K 480 -37 %, K 1536 -24 %, K 2048 -8 %; N 2592 K 1600 -11 %;
      // N 5120 K 1024 -25 %, K 1600 -9 %, K 2560 -1 %, K 3072 +9 % (the 4-stage ring)
      CUtensorMap th;
      uint64_t hd[2] = {(uint64_t)N, (uint64_t)M};
      uint64_t hs[1] = {(uint64_t)epi->ldc * 4};
      uint32_t hbox[2] = {32, 32};
      int rc = make_tmap_f32(&th, epi->out, 2, hd, hs, hbox);
      if (rc) return rc;
      return launch_gemm_pair<2, true, false, true>(ta, tb, p, s, &th);
    }
    if (staged && K <= 2048 && epg2) return launch_gemm_pair<2, true, true>(ta, tb, p, s);
    if (staged) return epg2 ? launch_gemm_pair<2, true>(ta, tb, p, s) : launch_gemm_pair<1, true>(ta, tb, p, s);
    return epg2 ? launch_gemm_pair<2, false>(ta, tb, p, s) : launch_gemm_pair<1, false>(ta, tb, p, s);
  }
  if (BN == 64) return epg2 ? launch_gemm<64, 2>(ta, tb, p, s) : launch_gemm<64, 1>(ta, tb, p, s);
  if (BN == 128) return epg2 ? launch_gemm<128, 2>(ta, tb, p, s) : launch_gemm<128, 1>(ta, tb, p, s);
  return epg2 ? launch_gemm<256, 2>(ta, tb, p, s) : launch_gemm<256, 1>(ta, tb, p, s);
}
