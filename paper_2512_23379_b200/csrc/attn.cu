// Attention kernels: softmax(Q K^T * scale) V per head, bidirectional (no mask
// beyond the key length). Restates the reference's mha_forward core
// (backends/reference.py:77-92; Cython row loop _fast.pyx:162-209).
//
//  (0) fmha2_tc_kernel — tcgen05 flash attention for long sequences, head_dim 64|128
//      (two 128-query tiles per CTA, P in TMEM; see the kernel's comment).
//  (3) xattn_tc_kernel  — short-KV tcgen05 kernel (Lk <= 128, one exact key block).
//  (1) attn_small_kernel — CUDA-core online-softmax kernel for short key sets
//      (cross-attention over conditioning tokens, ftlk-mode 9-token chunks).
#include <math.h>


#include "common.cuh"
#include "ftb_internal.h"

namespace ftb {

struct AttnParams {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;
  long long ldq, ldk, ldv, ldo;
  int Lq, Lk, heads, hd;
  float scale_log2;  // scale * log2(e)
  // Ulysses scatter epilogue (n_peers > 0): output row r goes to rank r / peer_rows,
  // row r % peer_rows of that rank's buffer (a peer-mapped pointer over NVLink)
  int n_peers;
  long long peer_rows;
  __nv_bfloat16* o_peers[FTB_MAX_PEERS];
  // fmha2 1-D grid: item = (head, 256-query block), n_qblk blocks per head. With ws != null
  // the items from split_first on (the partial last round) run as two CTAs each, one per half
  // of the key blocks, storing unnormalised fp32 O + (m, l) per row into ws for
  // fmha2_combine_kernel.
  int n_qblk, split_first;
  float* ws;
};

#ifdef FTB_FMHA_TIMELINE
// debug builds only: per-block clock64 stamps of the softmax warps of one CTA
__device__ long long g_fmha_tl[2][128][8];
#define FTB_TL(t, j, k)                                                                          \
  do {                                                                                           \
    if (blockIdx.x == 10 && blockIdx.y == 0 && (warp & 3) == 0 && lane == 0 && (j) < 128)          \
      g_fmha_tl[t][j][k] = clock64();                                                            \
  } while (0)
#else
#define FTB_TL(t, j, k) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ __nv_bfloat16* attn_out_row(const AttnParams& p, long long row) {
  if (p.n_peers) {
    const long long d = row / p.peer_rows;
    return p.o_peers[d] + (row - d * p.peer_rows) * p.ldo;
  }
  return p.o + row * p.ldo;
}

// ============================================================ tcgen05 flash kernel v2 (2 Q tiles / CTA)
// One CTA = one head x 256 queries as two 128-row tiles. The MMA warp interleaves the
// tiles — PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) — so the tensor core works on one tile
// while the other tile's softmax warpgroup (4 warps, one thread per row) runs. K and V
// blocks stream through a 3-slot TMA ring; half of the exponentials are evaluated with a
// degree-3 polynomial on the FMA pipe to offload MUFU (P is stored as bf16 anyway).
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;            // 1.5 * 2^23: round-to-nearest integer in the mantissa
  const float n = t - 12582912.f;
  const float f = x - n;                     // [-0.5, 0.5]
  float p = fmaf(f, 0.0555041086648216f, 0.2402265069591007f);
  p = fmaf(p, f, 0.6931471805599453f);
  p = fmaf(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (int)((unsigned)(__float_as_int(t) - 0x4B400000) << 23));
}

template <int HD>
struct Fmha2Cfg {
  static constexpr int BOX = 128 * 64 * 2;               // 128 rows x 64 cols bf16
  static constexpr int NBOX = HD / 64;
  static constexpr int TILE = NBOX * BOX;                // 128 rows x HD
  static constexpr int SLOTS = (HD == 128) ? 4 : 6;      // K/V ring depth
  static constexpr int OFF_Q = 0;                        // 2 tiles
  static constexpr int OFF_KV = OFF_Q + 2 * TILE;
  static constexpr int OFF_BAR = OFF_KV + SLOTS * TILE;
  static constexpr int SMEM = OFF_BAR + 512 + 1024;
};

// TMEM map (512 columns): S_t fp32 at [128t, 128t+128) with P_t (bf16 pairs) aliased onto
// its first 64 columns; O_t fp32 at [256 + 128t, 256 + 128t + HD).
// The softmax hands P over in two 64-key halves so PV of the first half overlaps the
// exponentials of the second (shortens the S -> softmax -> PV -> S chain).
template <int HD>
__global__ void __launch_bounds__(384, 1)
    fmha2_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using C = Fmha2Cfg<HD>;
  constexpr int NS = C::SLOTS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;         // [NS]
  uint64_t* kv_empty = bars + 1 + NS;   // [NS]
  uint64_t* s_full = bars + 1 + 2 * NS; // [2] per tile
  uint64_t* p_full = s_full + 2;        // [2]
  uint64_t* o_done = s_full + 4;        // [2]
  uint64_t* p_lo = s_full + 6;          // [2] first P half written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 8);

  const int warp = warp_id(), lane = lane_id();
  int item = blockIdx.x, part = -1;  // part >= 0: this CTA runs half of the key blocks
  if (p.ws && item >= p.split_first) {
    part = (item - p.split_first) & 1;
    item = p.split_first + ((item - p.split_first) >> 1);
  }
  const int qblk = item % p.n_qblk, head = item / p.n_qblk;
  const int n_kv_all = (p.Lk + 127) / 128;
  const int j0 = part == 1 ? n_kv_all / 2 : 0;                 // first global key block
  const int n_kv = part == 0 ? n_kv_all / 2 : n_kv_all - j0;  // key blocks of this CTA (loops count locally)

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 4);
      mbar_init(&p_lo[t], 4);
      mbar_init(&o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Register budget: the producer / MMA warpgroup gives registers to the two softmax
  // warpgroups (128*96 + 256*200 <= 384*168: inc blocks until the pool has them), which keeps a whole 128-column S row resident.
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;\n" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      const int col0 = head * HD;
      mbar_arrive_expect_tx(q_full, 2 * C::TILE);
      for (int t = 0; t < 2; ++t)
        for (int b = 0; b < C::NBOX; ++b)
          tma_load_2d(smem + C::OFF_Q + t * C::TILE + b * C::BOX, &tmQ, q_full, col0 + 64 * b, qblk * 256 + t * 128);
      for (int i = 0; i < 2 * n_kv; ++i) {  // item 2j = K_j, 2j+1 = V_j
        const int slot = i % NS;
        mbar_wait(&kv_empty[slot], ((i / NS) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[slot], C::TILE);
        const CUtensorMap* tm = (i & 1) ? &tmV : &tmK;
        for (int b = 0; b < C::NBOX; ++b)
          tma_load_2d(smem + C::OFF_KV + slot * C::TILE + b * C::BOX, tm, &kv_full[slot], col0 + 64 * b,
                      (j0 + (i >> 1)) * 128);
      }
    }
  } else if (warp == 1) {
    {  // warp-converged issue loop: one elected lane issues each tcgen05 op
      __syncwarp();
      constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16(128, HD, 0, 1);
      auto wait_item = [&](int i) { mbar_wait(&kv_full[i % NS], (i / NS) & 1); };
      auto issue_s = [&](int t, int j) {
        const uint32_t sq = smem_u32(smem + C::OFF_Q + t * C::TILE);
        const uint32_t sk = smem_u32(smem + C::OFF_KV + ((2 * j) % NS) * C::TILE);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * C::BOX + (kk & 3) * 32;
          mma_bf16_ss_elect(tmem + t * 128, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(sk + off, 16, 1024), idesc_s,
                      kk > 0);
        }
        mma_commit_elect(&s_full[t]);
      };
      auto issue_pv_part = [&](int t, int j, int k0, int k1) {  // O_t += P_t (TMEM) . V_j (smem, MN-major)
        const uint32_t sv = smem_u32(smem + C::OFF_KV + ((2 * j + 1) % NS) * C::TILE);
#pragma unroll
        for (int kk = k0; kk < k1; ++kk) {
          const uint64_t bd = sdesc_sw128(sv + kk * 16 * 128, C::BOX, 1024);
          mma_bf16_ts_elect(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, bd, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int t, int j) {
        mbar_wait(&p_lo[t], j & 1);
        tc_fence_after();
        issue_pv_part(t, j, 0, 4);
        mbar_wait(&p_full[t], j & 1);
        tc_fence_after();
        issue_pv_part(t, j, 4, 8);
        mma_commit_elect(&o_done[t]);
      };
      mbar_wait(q_full, 0);
      wait_item(0);
      tc_fence_after();
      issue_s(0, 0);
      issue_s(1, 0);
      mma_commit_elect(&kv_empty[0]);  // K_0 consumed by both tiles
      // Per block: PV_0(j), S_0(j+1), PV_1(j), S_1(j+1). S_t(j+1) overwrites the TMEM that
      // holds P_t(j), so it is issued after PV_t(j) (tcgen05 ops of a CTA execute in order).
      for (int j = 0; j < n_kv; ++j) {
        wait_item(2 * j + 1);  // V_j
        issue_pv(0, j);
        if (j + 1 < n_kv) {
          wait_item(2 * j + 2);  // K_{j+1}
          issue_s(0, j + 1);
        }
        issue_pv(1, j);
        mma_commit_elect(&kv_empty[(2 * j + 1) % NS]);  // V_j consumed
        if (j + 1 < n_kv) {
          issue_s(1, j + 1);
          mma_commit_elect(&kv_empty[(2 * j + 2) % NS]);  // K_{j+1} consumed by both tiles
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    const int t = (warp - 4) >> 2;  // tile handled by this warpgroup
    const int qw = warp & 3;
    const int row = qw * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qw * 32) << 16;
    const uint32_t tS = tmem + lane_off + t * 128;
    const uint32_t tO = tmem + lane_off + 256 + t * 128;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      FTB_TL(t, j, 0);
      mbar_wait(&s_full[t], j & 1);
      FTB_TL(t, j, 1);
      tc_fence_after();
#ifdef FTB_FMHA_NOSOFTMAX   // debug: MMA / TMA pipeline alone (the hand-off without any softmax work)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&p_lo[t]);
        mbar_arrive(&p_full[t]);
      }
      continue;
#endif
      uint32_t sr[128];
      tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(sr + 0));
      tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(sr + 64));
      tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(sr + 96));
      tmem_ld_wait();
      FTB_TL(t, j, 2);
      const int valid = p.Lk - (j0 + j) * 128;  // global key block
      if (valid < 128) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= valid) sr[c] = __float_as_uint(-INFINITY);
      }
      float mm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mm[u] = fmaxf(__uint_as_float(sr[2 * u]), __uint_as_float(sr[2 * u + 1]));
#pragma unroll
      for (int c = 16; c < 128; c += 16)   // 8 independent FMNMX3 chains (latency), 7 deep
#pragma unroll
        for (int u = 0; u < 8; ++u) mm[u] = fmax3(mm[u], __uint_as_float(sr[c + 2 * u]), __uint_as_float(sr[c + 2 * u + 1]));
      const float mx = fmaxf(fmax3(mm[0], mm[1], mm[2]), fmax3(mm[3], mm[4], fmax3(mm[5], mm[6], mm[7]))) * p.scale_log2;
      float m_use = m_ref;
      bool rescale = false;
      if (j == 0) {
        m_use = mx;
      } else if (mx > m_ref + 8.f) {
        m_use = mx;
        rescale = true;
      }
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
      const float2 nm2 = make_float2(-m_use, -m_use);
      float2 rs2 = make_float2(0.f, 0.f);
      // P_t (bf16 pairs) overwrites the first 64 columns of S_t: pack in place in sr[0..63]
      auto exp_chunks = [&](int ch0, int ch1) {
#pragma unroll
        for (int ch = ch0; ch < ch1; ++ch) {
          float2 e[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float2 x = ffma2(make_float2(__uint_as_float(sr[ch * 8 + 2 * u]), __uint_as_float(sr[ch * 8 + 2 * u + 1])),
                             sc2, nm2);
            if (u == 3) {  // one pair in four on the FMA pipe (offloads MUFU; 0 or 1/2 measured slower)
              x.x = fmaxf(x.x, -126.f);
              x.y = fmaxf(x.y, -126.f);
              e[u] = ex2_poly2(x);
            } else {
              e[u] = make_float2(ex2(x.x), ex2(x.y));
            }
            rs2 = fadd2(rs2, e[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) sr[ch * 4 + u] = pack_bf16(e[u].x, e[u].y);
        }
      };
      auto rescale_o = [&]() {
        if (__any_sync(0xffffffffu, rescale)) {
          const float f = rescale ? ex2(m_ref - m_use) : 1.f;
          l *= f;
#pragma unroll 1
          for (int c0 = 0; c0 < HD; c0 += 32) {
            uint32_t o[32];
            tmem_ld32(tO + c0, o);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 32; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * f);
            tmem_st32(tO + c0, o);
          }
        }
      };
      FTB_TL(t, j, 3);
      exp_chunks(0, 8);
      FTB_TL(t, j, 4);
      // PV_t(j-1) is complete here: the MMA warp committed s_full_t(j) after issuing PV_t(j-1),
      // and a commit tracks every earlier tcgen05 op of the thread, so O_t is stable and the
      // P region free without waiting on o_done
      FTB_TL(t, j, 5);
      tc_fence_after();
      rescale_o();
      tmem_st32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(sr + 0));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_lo[t]);
      exp_chunks(8, 16);
      tmem_st32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
      tmem_st_wait();
      FTB_TL(t, j, 6);
      l += rs2.x + rs2.y;
      m_ref = m_use;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[t]);
    }
    mbar_wait(&o_done[t], (n_kv - 1) & 1);
    tc_fence_after();
    const int grow = qblk * 256 + t * 128 + row;
    const float inv = 1.f / l;
    if (p.ws && (int)blockIdx.x >= p.split_first) {  // half of the keys: unnormalised O, (m_ref, l) for the combine
      float* ws = p.ws + (size_t)(blockIdx.x - p.split_first) * (256 * HD + 512);
      float4* wrow = reinterpret_cast<float4*>(ws + (size_t)(t * 128 + row) * HD);
#pragma unroll 1
      for (int c0 = 0; c0 < HD; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tO + c0, o);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 8; ++u)
          wrow[c0 / 4 + u] = make_float4(__uint_as_float(o[4 * u]), __uint_as_float(o[4 * u + 1]),
                                         __uint_as_float(o[4 * u + 2]), __uint_as_float(o[4 * u + 3]));
      }
      reinterpret_cast<float2*>(ws + 256 * HD)[t * 128 + row] = make_float2(m_ref, l);
    } else
#pragma unroll 1
    for (int c0 = 0; c0 < HD; c0 += 32) {
      uint32_t o[32];
      tmem_ld32(tO + c0, o);
      tmem_ld_wait();
      if (grow < p.Lq) {
        uint4* dst = reinterpret_cast<uint4*>(attn_out_row(p, grow) + head * HD + c0);
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(o[8 * qq + 0]) * inv, __uint_as_float(o[8 * qq + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(o[8 * qq + 2]) * inv, __uint_as_float(o[8 * qq + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(o[8 * qq + 4]) * inv, __uint_as_float(o[8 * qq + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(o[8 * qq + 6]) * inv, __uint_as_float(o[8 * qq + 7]) * inv);
          dst[qq] = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ============================================================ short-KV tcgen05 kernel
// Cross-attention of the wan DiT: 10 530 queries against Lk <= 128 conditioning keys
// (37 at the 14B shape). One key block, so the softmax is exact (no running max).
// Persistent CTAs (two per SM: 256 TMEM columns, < 100 KB smem each) walk a contiguous
// run of (head, query tile) items, so K/V (NKP = roundup(Lk, 16) rows) reload only when
// the head changes; Q of item k+1 loads while item k computes, and the MMA warp issues
// S(k+1) while the epilogue of item k drains O, so the kernel streams at the HBM rate of
// reading Q and writing O. TMEM: S/P [0,128) (P bf16 pairs aliased on S), O [128, 128+HD).
// The epilogue stages the bf16 O tile in the item's (consumed) Q slot and warp 3 writes it
// with TMA stores, so HBM sees full-line writes (TSTORE; the Ulysses scatter epilogue
// keeps per-row stores).
template <int HD>
struct XattnCfg {
  static constexpr int QBOX = 128 * 64 * 2;
  static constexpr int NBOX = HD / 64;
  static constexpr int QTILE = NBOX * QBOX;
  static constexpr int KVBOX = 128 * 64 * 2;          // sized for NKP <= 128
  static constexpr int KVTILE = NBOX * KVBOX;
  static constexpr int OFF_Q = 0;                     // [2] Q tiles
  static constexpr int OFF_K = OFF_Q + 2 * QTILE;
  static constexpr int OFF_V = OFF_K + KVTILE;
  static constexpr int OFF_BAR = OFF_V + KVTILE;
  static constexpr int SMEM_MAX = OFF_BAR + 256 + 1024;
};

template <int HD, int KMAX, bool TSTORE>
__global__ void __launch_bounds__(256, KMAX == 64 ? 2 : 1)
    xattn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const AttnParams p, int nkp, int n_qt) {
  using C = XattnCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kvbox = nkp * 128;                        // bytes of one 64-column K/V box
  const int kvtile = C::NBOX * kvbox;
  uint8_t* sQ = smem + C::OFF_Q;
  uint8_t* sK = sQ + 2 * C::QTILE;
  uint8_t* sV = sK + kvtile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kvtile);
  uint64_t* in_full = bars + 0;   // [2] Q tile
  uint64_t* in_empty = bars + 2;  // [2]
  uint64_t* s_full = bars + 4;
  uint64_t* p_full = bars + 5;
  uint64_t* o_full = bars + 6;
  uint64_t* o_free = bars + 7;
  uint64_t* kv_full = bars + 8;   // K/V of the current head
  uint64_t* kv_empty = bars + 9;
  uint64_t* staged = bars + 10;   // [2] O tile of slot b written to smem (TSTORE)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = warp_id(), lane = lane_id();
  const long long n_items = (long long)n_qt * p.heads;
  const int first = (int)(n_items * blockIdx.x / gridDim.x);
  const int last = (int)(n_items * (blockIdx.x + 1) / gridDim.x);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&in_full[b], 1);
      mbar_init(&in_empty[b], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    mbar_init(o_free, 4);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(&staged[0], 4);
    mbar_init(&staged[1], 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int k = 0, hk = 0, cur = -1;
      for (int it = first; it < last; ++it, ++k) {
        const int b = k & 1;
        const int head = it / n_qt, qt = it - head * n_qt;
        if (head != cur) {  // new head: K/V reload once the previous head's PVs are done
          mbar_wait(kv_empty, (hk & 1) ^ 1);
          mbar_arrive_expect_tx(kv_full, 2 * kvtile);
          for (int x = 0; x < C::NBOX; ++x) {
            tma_load_2d(sK + x * kvbox, &tmK, kv_full, head * HD + 64 * x, 0);
            tma_load_2d(sV + x * kvbox, &tmV, kv_full, head * HD + 64 * x, 0);
          }
          cur = head;
          ++hk;
        }
        mbar_wait(&in_empty[b], ((k >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&in_full[b], C::QTILE);
        for (int x = 0; x < C::NBOX; ++x)
          tma_load_2d(sQ + b * C::QTILE + x * C::QBOX, &tmQ, &in_full[b], head * HD + 64 * x, qt * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16(128, nkp, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16(128, HD, 0, 1);
      int k = 0, hk = 0, cur = -1;
      for (int it = first; it < last; ++it, ++k) {
        const int b = k & 1;
        const int head = it / n_qt;
        if (head != cur) {
          mbar_wait(kv_full, hk & 1);
          cur = head;
          ++hk;
        }
        mbar_wait(&in_full[b], (k >> 1) & 1);
        // S(k) overwrites P(k-1): ordered after PV(k-1) on the tensor pipe; the softmax
        // of item k-1 finished with S before it wrote P (p_full), which PV(k-1) waited on.
        tc_fence_after();
        const uint32_t sq = smem_u32(sQ + b * C::QTILE), sk = smem_u32(sK);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t offq = (kk >> 2) * C::QBOX + (kk & 3) * 32;
          const uint32_t offk = (kk >> 2) * kvbox + (kk & 3) * 32;
          mma_bf16_ss(tmem, sdesc_sw128(sq + offq, 16, 1024), sdesc_sw128(sk + offk, 16, 1024), idesc_s, kk > 0);
        }
        mma_commit(s_full);
        mbar_wait(p_full, k & 1);
        if (k > 0) mbar_wait(o_free, (k - 1) & 1);   // epilogue of item k-1 has read O
        tc_fence_after();
        const uint32_t sv = smem_u32(sV);
        for (int kk = 0; kk < nkp / 16; ++kk) {
          const uint64_t bd = sdesc_sw128(sv + kk * 16 * 128, kvbox, 1024);
          mma_bf16_ts(tmem + 128, tmem + kk * 8, bd, idesc_o, kk > 0 ? 1u : 0u);
        }
        mma_commit(o_full);
        if (!TSTORE) mma_commit(&in_empty[b]);   // TSTORE: freed by the store warp
        if (it + 1 == last || (it + 1) / n_qt != head) mma_commit(kv_empty);  // head done with K/V
      }
    }
  } else if (warp == 3) {
    if (TSTORE && lane == 0) {
      int k = 0;
      for (int it = first; it < last; ++it, ++k) {
        const int b = k & 1;
        const int head = it / n_qt, qt = it - head * n_qt;
        mbar_wait(&staged[b], (k >> 1) & 1);
        for (int x = 0; x < C::NBOX; ++x) tma_store_2d(&tmO, sQ + b * C::QTILE + x * C::QBOX, head * HD + 64 * x, qt * 128);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(&in_empty[b]);   // slot b may take the Q tile of item k+2
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (warp >= 4) {
    const int qw = warp & 3;
    const int row = qw * 32 + lane;
    const uint32_t lane_off = (uint32_t)(qw * 32) << 16;
    const uint32_t tS = tmem + lane_off, tO = tmem + lane_off + 128;
    int k = 0;
    for (int it = first; it < last; ++it, ++k) {
      const int head = it / n_qt, qt = it - head * n_qt;
      mbar_wait(s_full, k & 1);
      tc_fence_after();
      uint32_t sr[KMAX];
#pragma unroll
      for (int c = 0; c < KMAX / 32; ++c)
        if (c * 32 < nkp) tmem_ld32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
      tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < p.Lk) mx = fmaxf(mx, __uint_as_float(sr[c]));
      mx *= p.scale_log2;
      float l = 0.f;
#pragma unroll
      for (int c = 0; c < KMAX; c += 2) {
        if (c < nkp) {
          const float e0 = c < p.Lk ? ex2(fmaf(__uint_as_float(sr[c]), p.scale_log2, -mx)) : 0.f;
          const float e1 = c + 1 < p.Lk ? ex2(fmaf(__uint_as_float(sr[c + 1]), p.scale_log2, -mx)) : 0.f;
          l += e0 + e1;
          sr[c >> 1] = pack_bf16(e0, e1);
        }
      }
#pragma unroll
      for (int c = 0; c < KMAX / 64; ++c)
        if (c * 64 < nkp) tmem_st32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(sr + c * 32));
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      mbar_wait(o_full, k & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      const long long grow = (long long)qt * 128 + row;
      if (TSTORE) {
        uint8_t* stg = sQ + (k & 1) * C::QTILE + row * 128;
#pragma unroll 1
        for (int c0 = 0; c0 < HD; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(tO + c0, o);
          tmem_ld_wait();
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(o[8 * q8 + 0]) * inv, __uint_as_float(o[8 * q8 + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(o[8 * q8 + 2]) * inv, __uint_as_float(o[8 * q8 + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(o[8 * q8 + 4]) * inv, __uint_as_float(o[8 * q8 + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(o[8 * q8 + 6]) * inv, __uint_as_float(o[8 * q8 + 7]) * inv);
            const int c16 = ((c0 & 63) >> 3) + q8;   // 16-byte chunk within the 128-byte row
            *reinterpret_cast<uint4*>(stg + (c0 >> 6) * C::QBOX + ((c16 ^ (row & 7)) << 4)) = w;
          }
        }
      } else {
        __nv_bfloat16* orow = attn_out_row(p, grow < p.Lq ? grow : 0) + head * HD;
#pragma unroll 1
        for (int c0 = 0; c0 < HD; c0 += 32) {
          uint32_t o[32];
          tmem_ld32(tO + c0, o);
          tmem_ld_wait();
          if (grow < p.Lq) {
            uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(o[8 * q8 + 0]) * inv, __uint_as_float(o[8 * q8 + 1]) * inv);
              w.y = pack_bf16(__uint_as_float(o[8 * q8 + 2]) * inv, __uint_as_float(o[8 * q8 + 3]) * inv);
              w.z = pack_bf16(__uint_as_float(o[8 * q8 + 4]) * inv, __uint_as_float(o[8 * q8 + 5]) * inv);
              w.w = pack_bf16(__uint_as_float(o[8 * q8 + 6]) * inv, __uint_as_float(o[8 * q8 + 7]) * inv);
              dst[q8] = w;
            }
          }
        }
      }
      tc_fence_before();
      if (TSTORE) fence_proxy_async_smem();  // staged tile visible to the TMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(o_free);   // O drained: PV(k+1) may overwrite it
        if (TSTORE) mbar_arrive(&staged[k & 1]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<256>(tmem);
}

// Output columns the TMA store may touch: all heads of this call.
static long long head_cols(const AttnParams& p) { return (long long)p.heads * p.hd; }

template <int HD>
static int launch_xattn(const AttnParams& p, cudaStream_t s) {
  using C = XattnCfg<HD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaSuccess;
    for (auto fn : {xattn_tc_kernel<HD, 64, true>, xattn_tc_kernel<HD, 128, true>, xattn_tc_kernel<HD, 64, false>,
                    xattn_tc_kernel<HD, 128, false>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_MAX);
    if (e != cudaSuccess) return set_cuda_error(e, "xattn smem attribute");
    configured = true;
  }
  const int nkp = (p.Lk + 15) & ~15;
  CUtensorMap tq, tk, tv;
  int rc;
  {
    uint64_t dims[2] = {(uint64_t)p.ldq, (uint64_t)p.Lq};
    uint64_t strides[1] = {(uint64_t)p.ldq * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = make_tmap_bf16(&tq, p.q, 2, dims, strides, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)p.ldk, (uint64_t)p.Lk};
    uint64_t strides[1] = {(uint64_t)p.ldk * 2};
    uint32_t box[2] = {64, (uint32_t)nkp};
    if ((rc = make_tmap_bf16(&tk, p.k, 2, dims, strides, box))) return rc;
  }
  {
    uint64_t dims[2] = {(uint64_t)p.ldv, (uint64_t)p.Lk};
    uint64_t strides[1] = {(uint64_t)p.ldv * 2};
    uint32_t box[2] = {64, (uint32_t)nkp};
    if ((rc = make_tmap_bf16(&tv, p.v, 2, dims, strides, box))) return rc;
  }
  CUtensorMap to{};
  const bool tstore = p.n_peers == 0;
  if (tstore) {
    uint64_t dims[2] = {(uint64_t)(head_cols(p)), (uint64_t)p.Lq};
    uint64_t strides[1] = {(uint64_t)p.ldo * 2};
    uint32_t box[2] = {64, 128};
    if ((rc = make_tmap_bf16(&to, p.o, 2, dims, strides, box))) return rc;
  }
  const int n_qt = (p.Lq + 127) / 128;
  const int items = n_qt * p.heads;
  const int smem = C::OFF_K + 2 * (C::NBOX * nkp * 128) + 256 + 1024;
  const int grid = items < 2 * sm_count() ? items : 2 * sm_count();
  if (tstore) {
    if (nkp <= 64)
      xattn_tc_kernel<HD, 64, true><<<grid, 256, smem, s>>>(tq, tk, tv, to, p, nkp, n_qt);
    else
      xattn_tc_kernel<HD, 128, true><<<grid, 256, smem, s>>>(tq, tk, tv, to, p, nkp, n_qt);
  } else {
    if (nkp <= 64)
      xattn_tc_kernel<HD, 64, false><<<grid, 256, smem, s>>>(tq, tk, tv, to, p, nkp, n_qt);
    else
      xattn_tc_kernel<HD, 128, false><<<grid, 256, smem, s>>>(tq, tk, tv, to, p, nkp, n_qt);
  }
  return check_launch("xattn_tc_kernel");
}

// ============================================================ short-KV CUDA-core kernel
// grid (ceil(Lq/16), heads), 128 threads: warp w owns query rows 4w..4w+3 of the block.
// HDMAX bounds the shared-memory tile; the head width itself is runtime (any hd <= HDMAX).
template <int HDMAX>
__global__ void __launch_bounds__(128) attn_small_kernel(const AttnParams p) {
  const int HD = p.hd;
  constexpr int TK = 32;  // one key per lane per tile
  constexpr int DPL = (HDMAX + 31) / 32;
  __shared__ float Ks[TK][HDMAX + 1];
  __shared__ float Vs[TK][HDMAX];
  __shared__ float Qs[16][HDMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int head = blockIdx.y;
  const int r0 = blockIdx.x * 16;
  for (int i = threadIdx.x; i < 16 * HD; i += 128) {
    const int r = i / HD, d = i - (i / HD) * HD;
    const int gr = r0 + r;
    Qs[r][d] = (gr < p.Lq) ? __bfloat162float(p.q[(long long)gr * p.ldq + head * HD + d]) : 0.f;
  }
  float m[4], l[4], acc[4][DPL];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    m[r] = -INFINITY;
    l[r] = 0.f;
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[r][i] = 0.f;
  }
  for (int k0 = 0; k0 < p.Lk; k0 += TK) {
    __syncthreads();
    for (int i = threadIdx.x; i < TK * HD; i += 128) {
      const int r = i / HD, d = i - (i / HD) * HD;
      const int gk = k0 + r;
      float kv = 0.f, vv = 0.f;
      if (gk < p.Lk) {
        kv = __bfloat162float(p.k[(long long)gk * p.ldk + head * HD + d]);
        vv = __bfloat162float(p.v[(long long)gk * p.ldv + head * HD + d]);
      }
      Ks[r][d] = kv;
      Vs[r][d] = vv;
    }
    __syncthreads();
    const int nk = min(TK, p.Lk - k0);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int lr = warp * 4 + r;
      float s0 = 0.f;
#pragma unroll 4
      for (int d = 0; d < HD; ++d) s0 += Qs[lr][d] * Ks[lane][d];
      s0 = (lane < nk) ? s0 * p.scale_log2 : -INFINITY;
      float mx = s0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float mn = fmaxf(m[r], mx);
      const float corr = ex2(m[r] - mn);
      const float p0 = ex2(s0 - mn);
      float ps = p0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      l[r] = l[r] * corr + ps;
      m[r] = mn;
#pragma unroll
      for (int i = 0; i < DPL; ++i) acc[r][i] *= corr;
      for (int j = 0; j < nk; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p0, j);
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          const int d = lane + 32 * i;
          if (d < HD) acc[r][i] += pj * Vs[j][d];
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gr = r0 + warp * 4 + r;
    if (gr >= p.Lq) continue;
    const float inv = 1.f / l[r];
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int d = lane + 32 * i;
      if (d < HD) attn_out_row(p, gr)[head * HD + d] = __float2bfloat16_rn(acc[r][i] * inv);
    }
  }
}

// Merge the two key halves of each split item: O = (O0 2^(m0-m) + O1 2^(m1-m)) / (l0 2^(m0-m) +
// l1 2^(m1-m)), m = max(m0, m1) (m in the kernel's log2 units), stored like fmha2's epilogue.
template <int HD>
__global__ void __launch_bounds__(256) fmha2_combine_kernel(const AttnParams p) {
  const int s = blockIdx.x, r = threadIdx.x;
  const int item = p.split_first + s;
  const int qblk = item % p.n_qblk, head = item / p.n_qblk;
  const long long grow = (long long)qblk * 256 + r;
  if (grow >= p.Lq) return;
  const float* w0 = p.ws + (size_t)(2 * s) * (256 * HD + 512);
  const float* w1 = w0 + (256 * HD + 512);
  const float2 a = reinterpret_cast<const float2*>(w0 + 256 * HD)[r];
  const float2 b = reinterpret_cast<const float2*>(w1 + 256 * HD)[r];
  const float m = fmaxf(a.x, b.x);
  const float f0 = exp2f(a.x - m), f1 = exp2f(b.x - m);
  const float inv = 1.f / (a.y * f0 + b.y * f1);
  const float g0 = f0 * inv, g1 = f1 * inv;
  const float4* o0 = reinterpret_cast<const float4*>(w0 + (size_t)r * HD);
  const float4* o1 = reinterpret_cast<const float4*>(w1 + (size_t)r * HD);
  uint4* dst = reinterpret_cast<uint4*>(attn_out_row(p, grow) + head * HD);
#pragma unroll 4
  for (int c = 0; c < HD / 8; ++c) {
    const float4 x0 = o0[2 * c], x1 = o0[2 * c + 1], y0 = o1[2 * c], y1 = o1[2 * c + 1];
    dst[c] = make_uint4(pack_bf16(x0.x * g0 + y0.x * g1, x0.y * g0 + y0.y * g1),
                        pack_bf16(x0.z * g0 + y0.z * g1, x0.w * g0 + y0.w * g1),
                        pack_bf16(x1.x * g0 + y1.x * g1, x1.y * g0 + y1.y * g1),
                        pack_bf16(x1.z * g0 + y1.z * g1, x1.w * g0 + y1.w * g1));
  }
}

// KV-split tail round: the R = items % SMs items of the partial last round run as two key halves
// each on otherwise idle SMs when 2R <= SMs (14B: 1680 items = 11.35 rounds -> 11.5; 1.3B: 3.4 ->
// 3.5). Returns R (0: no split) for this device's SM count.
static int fmha2_split_items(int Lq, int Lk, int heads) {
  const int items = ((Lq + 255) / 256) * heads;
  const int nsm = sm_count();
  const int R = items % nsm;
  return (items > nsm && R > 0 && 2 * R <= nsm && (Lk + 127) / 128 >= 4) ? R : 0;
}

static size_t fmha2_ws_bytes(int R, int hd) { return (size_t)2 * R * (256 * hd + 512) * sizeof(float); }

template <int HD>
static int launch_fmha2(const AttnParams& p_in, cudaStream_t s, float* ws, size_t ws_bytes) {
  AttnParams p = p_in;
  using C = Fmha2Cfg<HD>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(fmha2_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return set_cuda_error(e, "fmha2 smem attribute");
    configured = true;
  }
  CUtensorMap tq, tk, tv;
  auto mk = [&](CUtensorMap* m, const void* ptr, long long ld, int rows) {
    uint64_t dims[2] = {(uint64_t)ld, (uint64_t)rows};
    uint64_t strides[1] = {(uint64_t)ld * 2};
    uint32_t box[2] = {64, 128};
    return make_tmap_bf16(m, ptr, 2, dims, strides, box);
  };
  int rc;
  if ((rc = mk(&tq, p.q, p.ldq, p.Lq))) return rc;
  if ((rc = mk(&tk, p.k, p.ldk, p.Lk))) return rc;
  if ((rc = mk(&tv, p.v, p.ldv, p.Lk))) return rc;
  // 1-D grid of (head, query block) items, query block fastest (CTAs running together share
  // K/V in L2); the partial last round splits over the keys when the caller's workspace holds it
  p.n_qblk = (p.Lq + 255) / 256;
  const int items = p.n_qblk * p.heads;
  const int R = fmha2_split_items(p.Lq, p.Lk, p.heads);
  p.ws = nullptr;
  p.split_first = items;
  if (R && ws && ws_bytes >= fmha2_ws_bytes(R, HD)) {
    p.ws = ws;
    p.split_first = items - R;
  }
  const int grid = p.ws ? items + R : items;
  fmha2_tc_kernel<HD><<<grid, 384, C::SMEM, s>>>(tq, tk, tv, p);
  rc = check_launch("fmha2_tc_kernel");
  if (rc || !p.ws) return rc;
  fmha2_combine_kernel<HD><<<R, 256, 0, s>>>(p);
  return check_launch("fmha2_combine_kernel");
}

template <int HDMAX>
static int launch_small(const AttnParams& p, cudaStream_t s) {
  dim3 grid((p.Lq + 15) / 16, p.heads);
  attn_small_kernel<HDMAX><<<grid, 128, 0, s>>>(p);
  return check_launch("attn_small_kernel");
}

// Attention probabilities for the reference mha_forward cache (backends/reference.py:86-88):
// one CTA per (query r, head h); scores for every key into smem-free registers/global, row max
// and sum by block reduction, then the normalised row. Any Lk; head_dim <= 256 (q row in smem).
__global__ void __launch_bounds__(128) attn_probs_kernel(const __nv_bfloat16* __restrict__ q, long long ldq,
                                                         const __nv_bfloat16* __restrict__ k, long long ldk, int Lq,
                                                         int Lk, int hd, float scale, float* __restrict__ p) {
  __shared__ float qs[256];
  __shared__ float red[4];
  const int r = blockIdx.x, h = blockIdx.y;
  for (int d = threadIdx.x; d < hd; d += 128) qs[d] = __bfloat162float(q[(long long)r * ldq + h * hd + d]);
  __syncthreads();
  float* prow = p + ((long long)h * Lq + r) * Lk;
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < Lk; j += 128) {
    const __nv_bfloat16* kr = k + (long long)j * ldk + h * hd;
    float s = 0.f;
    for (int d = 0; d < hd; ++d) s = fmaf(qs[d], __bfloat162float(kr[d]), s);
    s *= scale;
    prow[j] = s;
    mx = fmaxf(mx, s);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < Lk; j += 128) {
    const float e = expf(prow[j] - mx);
    prow[j] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  const float inv = 1.f / ((red[0] + red[1]) + (red[2] + red[3]));
  for (int j = threadIdx.x; j < Lk; j += 128) prow[j] *= inv;
}

}  // namespace ftb

using namespace ftb;

static int attention_run(int32_t impl, AttnParams& p, float* ws, size_t ws_bytes, void* stream) {
  const long long ldq = p.ldq, ldk = p.ldk, ldv = p.ldv, ldo = p.ldo;
  const int head_dim = p.hd;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (impl == 3) {  // short-KV tcgen05 kernel (Lk <= 128)
    if ((ldq & 7) || (ldk & 7) || (ldv & 7) || (ldo & 7)) return set_error(FTB_EINVAL, "xattn: ld alignment");
    if (p.Lk > 128) return set_error(FTB_EINVAL, "xattn: Lk must be <= 128");
    if (head_dim == 128) return launch_xattn<128>(p, s);
    if (head_dim == 64) return launch_xattn<64>(p, s);
    return set_error(FTB_EINVAL, "xattn: head_dim must be 64 or 128");
  }
  if (impl == 0) {  // flash kernel: 2 Q tiles per CTA, two softmax warpgroups
    if ((ldq & 7) || (ldk & 7) || (ldv & 7) || (ldo & 7)) return set_error(FTB_EINVAL, "fmha: ld alignment");
    if (head_dim == 128) return launch_fmha2<128>(p, s, ws, ws_bytes);
    if (head_dim == 64) return launch_fmha2<64>(p, s, ws, ws_bytes);
    return set_error(FTB_EINVAL, "fmha: head_dim must be 64 or 128");
  }
  if (impl != 1) return set_error(FTB_EINVAL, "attention: impl must be 0 (flash), 1 (CUDA-core) or 3 (short KV)");
  if (head_dim <= 16) return launch_small<16>(p, s);
  if (head_dim <= 32) return launch_small<32>(p, s);
  if (head_dim <= 64) return launch_small<64>(p, s);
  if (head_dim <= 128) return launch_small<128>(p, s);
  return set_error(FTB_EINVAL, "attention: head_dim must be <= 128");
}

static int default_impl(int Lq, int Lk, int head_dim) {
  if ((head_dim == 64 || head_dim == 128) && Lq >= 64) return Lk <= 128 ? 3 : 0;
  return 1;
}

extern "C" size_t ftb_attention_workspace_bytes(int32_t Lq, int32_t Lk, int32_t heads, int32_t head_dim) {
  if (Lq <= 0 || Lk <= 0 || heads <= 0 || default_impl(Lq, Lk, head_dim) != 0) return 0;
  const int R = fmha2_split_items(Lq, Lk, heads);
  return R ? fmha2_ws_bytes(R, head_dim) : 0;
}

extern "C" int ftb_attention_probs(const void* q, int64_t ldq, const void* k, int64_t ldk, int32_t Lq, int32_t Lk,
                                   int32_t heads, int32_t head_dim, float scale, float* p, void* stream) {
  if (!q || !k || !p || Lq < 0 || Lk <= 0 || heads <= 0 || head_dim <= 0 || head_dim > 256)
    return set_error(FTB_EINVAL, "attention_probs: bad arguments (head_dim must be in [1, 256])");
  if (ldq < (int64_t)heads * head_dim || ldk < (int64_t)heads * head_dim)
    return set_error(FTB_EINVAL, "attention_probs: ld smaller than heads * head_dim");
  if (Lq == 0) return FTB_OK;
  attn_probs_kernel<<<dim3(Lq, heads), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(q), ldq, static_cast<const __nv_bfloat16*>(k), ldk, Lq, Lk, head_dim, scale,
      p);
  return check_launch("attn_probs_kernel");
}

#ifdef FTB_FMHA_TIMELINE
extern "C" int ftb_debug_fmha_timeline(long long* out) {
  return cudaMemcpyFromSymbol(out, g_fmha_tl, sizeof(g_fmha_tl)) == cudaSuccess ? FTB_OK : FTB_ECUDA;
}
#endif

extern "C" int ftb_attention_impl(int32_t impl, const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                                  int64_t ldv, void* o, int64_t ldo, int32_t Lq, int32_t Lk, int32_t heads,
                                  int32_t head_dim, float scale, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  if (!q || !k || !v || !o || Lq < 0 || Lk <= 0 || heads <= 0 || head_dim <= 0)
    return set_error(FTB_EINVAL, "attention: bad arguments");
  if (Lq == 0) return FTB_OK;
  AttnParams p{};
  p.q = (const __nv_bfloat16*)q;
  p.k = (const __nv_bfloat16*)k;
  p.v = (const __nv_bfloat16*)v;
  p.o = (__nv_bfloat16*)o;
  p.ldq = ldq;
  p.ldk = ldk;
  p.ldv = ldv;
  p.ldo = ldo;
  p.Lq = Lq;
  p.Lk = Lk;
  p.heads = heads;
  p.hd = head_dim;
  p.scale_log2 = scale * 1.4426950408889634f;
  return attention_run(impl, p, (float*)workspace, workspace_bytes, stream);
}

extern "C" int ftb_attention_scatter(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                                     int64_t ldv, void* const* o_peers, int32_t n_peers, int64_t peer_rows,
                                     int64_t ldo, int32_t Lq, int32_t Lk, int32_t heads, int32_t head_dim,
                                     float scale, void* workspace, size_t workspace_bytes, void* stream) {
  if (!q || !k || !v || !o_peers || n_peers < 1 || n_peers > FTB_MAX_PEERS || peer_rows <= 0 || Lq < 0 || Lk <= 0 ||
      heads <= 0 || head_dim <= 0)
    return set_error(FTB_EINVAL, "attention_scatter: bad arguments");
  if ((long long)n_peers * peer_rows < Lq) return set_error(FTB_EINVAL, "attention_scatter: rows exceed peers");
  for (int i = 0; i < n_peers; ++i)
    if (!o_peers[i]) return set_error(FTB_EINVAL, "attention_scatter: null peer pointer");
  if (Lq == 0) return FTB_OK;
  AttnParams p{};
  p.q = (const __nv_bfloat16*)q;
  p.k = (const __nv_bfloat16*)k;
  p.v = (const __nv_bfloat16*)v;
  p.o = (__nv_bfloat16*)o_peers[0];
  p.ldq = ldq;
  p.ldk = ldk;
  p.ldv = ldv;
  p.ldo = ldo;
  p.Lq = Lq;
  p.Lk = Lk;
  p.heads = heads;
  p.hd = head_dim;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.n_peers = n_peers;
  p.peer_rows = peer_rows;
  for (int i = 0; i < n_peers; ++i) p.o_peers[i] = (__nv_bfloat16*)o_peers[i];
  return attention_run(default_impl(Lq, Lk, head_dim), p, (float*)workspace, workspace_bytes, stream);
}

extern "C" int ftb_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                             void* o, int64_t ldo, int32_t Lq, int32_t Lk, int32_t heads, int32_t head_dim,
                             float scale, void* workspace, size_t workspace_bytes, void* stream) {
  return ftb_attention_impl(default_impl(Lq, Lk, head_dim), q, ldq, k, ldk, v, ldv, o, ldo, Lq, Lk, heads, head_dim,
                            scale, workspace, workspace_bytes, stream);
}
