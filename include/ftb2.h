/*
 * ftb2 — C ABI of the B200 (sm_100a) streaming hot path.
 *
 * Plain pointers and sizes only: every buffer is a DEVICE pointer owned by the
 * caller (PyTorch caching allocator in the Python host); kernels never
 * allocate. `stream` is a cudaStream_t passed as void*. All entry points only
 * enqueue work (no implicit synchronisation) and are CUDA-graph capturable.
 * Return 0 on success or one of the FTB_E* codes; ftb_last_error() returns a
 * thread-local message. The Python host maps FTB_EINVAL -> ConfigError and
 * FTB_ENONFINITE -> NumericError (reference errors.py:4-18).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/ftlk):
 *   ftb_gemm_bf16 ........ backends/reference.py:17-18 dense_forward (x @ w + b), plus the
 *                          fused epilogues of net.py:230-274 (bias, GELU :266, residual
 *                          adds :256/:261/:268, embedding sum :232) and wan-mode AdaLN gates
 *   ftb_norm_modulate .... backends/reference.py:41-46 layernorm_forward (+ AdaLN modulation)
 *   ftb_attention ........ backends/reference.py:77-92 mha_forward core (softmax(QK^T/sqrt(hd))V),
 *                          self (net.py:254) and cross (net.py:259) attention
 *   ftb_gelu_bf16 ........ backends/reference.py:28-31 gelu_forward (standalone form)
 *   ftb_patchify_composite diffusion.py:133-135,150-179 composite assembly (Eq.1 channel stack)
 *   ftb_unpatch_ddim ..... diffusion.py:229-236 x0 slice + DDIM update; streaming.py:298-299 tail
 *   ftb_codec_decode ..... world.py:206-210 Codec.decode (latents @ Q)
 *   ftb_vae_* ............ wan-mode causal VAE decoder (build-defined)
 *   ftb_sym_* / ftb_ipc_* / ftb_peer_barrier / peer epilogues
 *                          Ulysses sequence parallel over NVLink peer memory (the
 *                          reference runs the DiT on one process, net.py:240-276)
 */
#ifndef FTB2_H
#define FTB2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTB_OK 0
#define FTB_EINVAL 1
#define FTB_ECUDA 2
#define FTB_ENCCL 3
#define FTB_ENONFINITE 4

#define FTB_MAX_PEERS 8          /* ranks of one NVLink domain addressed by a peer epilogue */
#define FTB_IPC_HANDLE_BYTES 64

int ftb_version(void);
const char* ftb_last_error(void);
int ftb_device_sm_count(int device);

/* ---------------------------------------------------------------- GEMM */
enum {
  FTB_EPI_BF16 = 0,       /* out_bf16 = acc + bias                                  */
  FTB_EPI_GELU_BF16 = 1,  /* out_bf16 = gelu_tanh(acc + bias)                       */
  FTB_EPI_F32 = 2,        /* out_f32  = acc + bias                                  */
  FTB_EPI_RESID_F32 = 3,  /* out_f32 += gate[g] * (acc + bias)   (gate NULL -> 1)   */
  FTB_EPI_ROWADD_F32 = 4, /* out_f32  = acc + bias + vec[g]                         */
  FTB_EPI_QKV_ROPE = 5,   /* bf16 q|k|v with 3D RoPE on q,k; Ulysses send layout    */
  FTB_EPI_SEG_SOFTMAX = 6 /* bf16 per-segment softmax of the logits (folded cross-attn) */
};

/* 3D rotary tables (wan mode): per-token float32 cos/sin [token][head_dim/2]
 * (token = row + row_offset, frame-major), composed on the host from the float64
 * per-axis tables (pairs [0,pt) frame axis, [pt,pt+ph) row axis, rest column axis). */
typedef struct ftb_rope3d {
  const float* cos_full;
  const float* sin_full;
} ftb_rope3d;

typedef struct ftb_epilogue {
  int32_t kind;
  int32_t rows_per_group;  /* g(row) = (row + row_offset) / rows_per_group */
  int64_t row_offset;
  const float* bias;       /* [N] or NULL */
  const float* group_vec;  /* [G][group_ld] gate / additive vector or NULL */
  int64_t group_ld;
  void* out;               /* bf16 or f32, [M][ldc] */
  int64_t ldc;
  /* FTB_EPI_QKV_ROPE only: column c of [0,3*heads*head_dim) -> (which, head, d);
   * stored at ((dest*M + row)*3 + which)*hpr*hd + (head%hpr)*hd + d, dest = head/hpr. */
  int32_t heads, head_dim, heads_per_rank;
  /* FTB_EPI_SEG_SOFTMAX reuses them: heads = segments S, head_dim = segment width J (multiple of
   * 8, <= 48), heads_per_rank = n_cond. GEMM column t*256 + s*J + j (s < 256/J) is key j of
   * segment t*(256/J) + s; out[row][seg*J + j] = softmax over j < n_cond (0 for j >= n_cond);
   * N = 256 * ceil(S / (256/J)). */
  const ftb_rope3d* rope;  /* NULL: no rotation */
  /* Peer stores (Ulysses over NVLink; 0 = local `out`):
   *  QKV_ROPE: n_peers = heads/heads_per_rank; head group `dest`'s block [M][3][hpr][hd]
   *            goes to peer_out[dest] (rank dest's receive buffer at this rank's slot);
   *  F32:      every peer_out[i] receives the full [M][ldc] result (fused all-gather). */
  int32_t n_peers;
  void* peer_out[FTB_MAX_PEERS];
  /* Block-diagonal operand (zero-initialise for a dense GEMM): band_k > 0 declares that row r
   * of A (band_side 0) or of B (band_side 1) is non-zero only in K columns [b*band_k,
   * (b+1)*band_k), b = (r / band_tile) * band_per_tile + (r % band_tile) / band_rows (band_tile 0:
   * b = r / band_rows). The CTA-pair kernel then runs each tile's K loop over the union of its
   * rows' bands only (the skipped products are exact zeros; the folded cross-attention's
   * At = blockdiag(K) . Wq^T and Bt = Wo^T . blockdiag(V)^T). */
  int32_t band_side, band_rows, band_tile, band_per_tile, band_k;
  /* Kernel selection of this call (0 = the product defaults; A/B benchmarks and tests set it):
   * bits 0-1: 0 auto (CTA pair when M, N >= 256), 1 single CTA, 2 CTA pair; +4 row-per-thread
   * residual epilogue of the pair kernel (instead of the smem-staged one); +8 no L2 prefetch of
   * the residual rows; +16 long-K residual GEMMs on one epilogue warpgroup; +32 no TMA-staged h
   * tiles for short-K (<= 2048) residual GEMMs. */
  int32_t variant;
  /* CTA-pair raster group (256-row m-blocks sharing one B sweep in L2): 0 auto (A panels of the
   * group ~40 MB, at least 8). */
  int32_t raster_group;
  /* Split-K tail wave of long-K residual GEMMs (K >= 8192): the partial last round's tiles run
   * as ordered K-slices on the idle CTA pairs, serialised through FTB_TAIL_COUNTER_WORDS u32
   * counters in device memory OWNED BY THE CALLER (zero-initialised once; every launch leaves
   * them zero). Launches sharing one counter buffer must be stream-ordered (one buffer per
   * stream of launches, e.g. per DeviceDenoiser). NULL: the tail runs unsplit. */
  uint32_t* tail_counters;
} ftb_epilogue;
#define FTB_TAIL_COUNTER_WORDS 2048

/* C[M,N] = A[M,K] . B[N,K]^T (bf16 in, fp32 accumulate, tcgen05 + TMEM, TMA-fed).
 * A is read as a_chunks K-slices of width K/a_chunks: element (r,k) at
 * A + (k / kc) * a_chunk_stride + r * lda + (k % kc) (Ulysses gather; a_chunks=1 plain).
 * Requirements: lda, ldb multiples of 8 elements; K/a_chunks multiple of 64 when a_chunks>1. */
int ftb_gemm_bf16(const void* A, int64_t lda, int32_t a_chunks, int64_t a_chunk_stride,
                  const void* B, int64_t ldb, int32_t M, int32_t N, int32_t K,
                  const ftb_epilogue* epi, void* stream);

/* ---------------------------------------------------------------- norms */
/* y = ((x - mean) * rstd) * (gamma?gamma:1) * (scale?1+scale[g]:1) + (beta?beta:0) + (shift?shift[g]:0)
 * rstd = 1/sqrt(var + eps), population variance; g = (row+row_offset)/rows_per_group.
 * Writes bf16 y [M][ldy]; optional f32 mean/rstd [M]. */
int ftb_norm_modulate(const float* x, int64_t ldx, int32_t M, int32_t N,
                      const float* gamma, const float* beta,
                      const float* scale, const float* shift, int64_t mod_ld,
                      int32_t rows_per_group, int64_t row_offset, float eps,
                      void* y, int64_t ldy, float* mean_out, float* rstd_out, void* stream);

/* ---------------------------------------------------------------- attention */
/* o[r, h*hd + d] = softmax_j(q_r . k_j * scale) v_j  per head h (bidirectional, no mask
 * beyond Lk). Row r of q at q + r*ldq + h*head_dim (bf16); same for k, v, o.
 * workspace: optional fp32 device scratch OWNED BY THE CALLER, workspace_bytes >=
 * ftb_attention_workspace_bytes(Lq, Lk, heads, head_dim) (0 when no split applies): the flash
 * kernel then runs the partial last round of (head, 256-query) items as two key halves on the
 * idle SMs plus a combine kernel. NULL or too small: every item runs whole (same results up to
 * fp32 rounding of the merge). Launches sharing one workspace must be stream-ordered. */
int ftb_attention(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                  void* o, int64_t ldo, int32_t Lq, int32_t Lk, int32_t heads, int32_t head_dim,
                  float scale, void* workspace, size_t workspace_bytes, void* stream);
/* Bytes of the KV-split workspace for this shape on the current device (0: no split). */
size_t ftb_attention_workspace_bytes(int32_t Lq, int32_t Lk, int32_t heads, int32_t head_dim);
/* Explicit kernel selection (tests / benchmarks): 0 = tcgen05 flash kernel (head_dim 64|128),
 * 1 = CUDA-core kernel (any head_dim <= 128), 3 = short-KV tcgen05 kernel (Lk <= 128). */
int ftb_attention_impl(int32_t impl, const void* q, int64_t ldq, const void* k, int64_t ldk,
                       const void* v, int64_t ldv, void* o, int64_t ldo, int32_t Lq, int32_t Lk,
                       int32_t heads, int32_t head_dim, float scale, void* workspace, size_t workspace_bytes,
                       void* stream);

/* The attention probabilities themselves, p[h][r][j] = softmax_j(q_r . k_j * scale) (fp32,
 * [heads][Lq][Lk] dense): the `p` entry of the reference's mha_forward cache
 * (backends/reference.py:86-88, returned at :92), which the flash kernels never materialise.
 * CUDA-core, one CTA per (query, head); any head_dim <= 256. For the drop-in backend table's
 * cache, not for the hot path. */
int ftb_attention_probs(const void* q, int64_t ldq, const void* k, int64_t ldk, int32_t Lq, int32_t Lk,
                        int32_t heads, int32_t head_dim, float scale, float* p, void* stream);

/* Ulysses all-to-all #2 fused into the epilogue: output row r is stored at row r % peer_rows
 * of o_peers[r / peer_rows] (device pointers, peer-mapped; host array of n_peers entries). */
int ftb_attention_scatter(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v, int64_t ldv,
                          void* const* o_peers, int32_t n_peers, int64_t peer_rows, int64_t ldo, int32_t Lq,
                          int32_t Lk, int32_t heads, int32_t head_dim, float scale, void* workspace,
                          size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- peer memory (multi-GPU) */
/* IPC-exportable zeroed device allocation / free. */
int ftb_sym_alloc(size_t bytes, void** ptr);
int ftb_sym_free(void* ptr);
/* cudaIpc handle of an ftb_sym_alloc pointer (FTB_IPC_HANDLE_BYTES bytes) and its import
 * into another process of the node (peer access enabled lazily); close undoes import. */
int ftb_ipc_export(const void* ptr, uint8_t* handle);
int ftb_ipc_import(const uint8_t* handle, void** ptr);
int ftb_ipc_close(void* ptr);
/* Stream-ordered device-to-device copy (peer-mapped destinations: VAE halo rows). */
int ftb_copy_d2d(void* dst, const void* src, size_t bytes, void* stream);
/* Stream-ordered strided device-to-device copy of `height` rows of `width` bytes (pitches in
 * bytes): a VAE row slab [T][rows][W][3] into rank 0's peer-mapped full frames [T][H][W][3]. */
int ftb_copy_d2d_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                    void* stream);
/* Stream-ordered barrier over `world` ranks: flags[i] = rank i's [world] u32 flag words
 * (peer-mapped), epoch = this rank's device counter (incremented per call, so the barrier
 * is CUDA-graph capturable). Fences prior stores system-wide, signals every rank, then
 * waits for all; traps after timeout_s seconds instead of hanging. */
int ftb_peer_barrier(uint32_t* const* flags, uint32_t* epoch, int32_t rank, int32_t world, double timeout_s,
                     void* stream);
/* Protocol self-test of ftb_peer_barrier with `world` concurrent ranks on one device (one
 * co-resident block per rank, cooperative launch): `rounds` x (payload store, barrier, check
 * every rank's payload, barrier). Caller-zeroed buffers: flags [world][world], epochs [world],
 * data [rounds][world]; errors[0] += mismatches. Used by the tests (one GPU emulates the ranks
 * without separate launches that wait on one another). */
int ftb_peer_barrier_selftest(int32_t world, int32_t rounds, uint32_t* flags, uint32_t* epochs, uint32_t* data,
                              uint32_t* errors, double timeout_s, void* stream);

/* Folded cross-attention (wan mode; the cond K/V are fixed for a chunk).
 * Block-diagonal operands for folding the cross-attention projections on the tensor cores
 * (net.py:259-261 composed with the chunk's fixed cond K/V): kbd[(h,j)][h*hd+d] = scale*K[j][h*hd+d],
 * vbd[(h,j)][h*hd+d] = V[j][h*hd+d], kv = [n_cond][K | V] bf16. Only the diagonal blocks are
 * written (caller zero-fills kbd / vbd once). Then At = kbd . Wq^T and Bt = Wo^T . vbd^T are two
 * ftb_gemm_bf16 calls. k_tile_segs > 0 puts kbd row (h,j) at (h / k_tile_segs) * 256 +
 * (h % k_tile_segs) * J + j: the FTB_EPI_SEG_SOFTMAX column order for the logits GEMM. */
int ftb_xattn_blockdiag(const void* kv, int64_t ldkv, int32_t n_cond, int32_t heads, int32_t head_dim, int32_t J,
                        float scale, void* kbd, void* vbd, int64_t ld, int32_t k_tile_segs, void* stream);

/* ---------------------------------------------------------------- elementwise */
int ftb_gelu_bf16(const void* x, void* y, int64_t n, void* stream);
int ftb_silu_f32_to_bf16(const float* x, void* y, int64_t n, void* stream);
int ftb_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream);
int ftb_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream);

/* Eq.1 composite -> patch tokens. motion [Lm][D][H][W], z [Lc-Lm][D][H][W],
 * reference [D][H][W] (f32). Token (f, y, x) = f*(H/ph)*(W/pw) + y*(W/pw) + x, feature
 * (c*ph + py)*pw + px over channels c in [z_noise(D) | z_mask(1) | z_cond(D)].
 * out bf16 [Lc*T][ldo], columns [in_features, ldo) zero-filled. */
int ftb_patchify_composite(const float* motion, const float* z, const float* reference,
                           int32_t Lm, int32_t Lc, int32_t D, int32_t H, int32_t W,
                           int32_t ph, int32_t pw, void* out, int64_t ldo, void* stream);

/* Same token layout from an arbitrary stacked composite f32 [Lc][C][H][W] (C = 2D+1 channels
 * z_noise | z_mask | z_cond as given: non-canonical masks / conditioning rows,
 * diffusion.py:89-135 CompositeInput, consumed by net.py:223-238). */
int ftb_patchify_stacked(const float* stacked, int32_t Lc, int32_t C, int32_t H, int32_t W, int32_t ph, int32_t pw,
                         void* out, int64_t ldo, void* stream);

/* x0 tokens f32 [Lc*T][ldx] (feature (c*ph+py)*pw+px) -> target frames.
 * x0_out [Lc-Lm][D][H][W] = x0 of frames >= Lm; if update:
 * z = a_n*x0 + s_n*(z - a_i*x0)/s_i (DDIM, diffusion.py:233-236). */
int ftb_unpatch_ddim(const float* x0_tok, int64_t ldx, int32_t Lm, int32_t Lc, int32_t D,
                     int32_t H, int32_t W, int32_t ph, int32_t pw, float* z, float* x0_out,
                     float a_i, float s_i, float a_n, float s_n, int32_t update, void* stream);

/* frames[n][D] = latents[n][D] @ Q[D][D]   (f32; orthogonal codec) */
int ftb_codec_decode(const float* latents, const float* Q, float* frames, int32_t n, int32_t D,
                     void* stream);

/* out[l][f][j] = a[f][j] + b[l][j], l < Lb, f < F, j < n (AdaLN tables). */
int ftb_add_bcast_f32(const float* a, int64_t F, int64_t n, const float* b, int64_t Lb, float* out, void* stream);

/* ---------------------------------------------------------------- VAE decoder (wan mode) */
/* Causal 3D conv as implicit GEMM (tcgen05): in bf16 [T_in][H][W][Cin] channel-last,
 * w_t bf16 [Cout][KT*KH*KW*Cin] (k = ((dt*KH+dy)*KW+dx)*Cin + c), stride 1, spatial
 * zero padding KH/2, KW/2; output frame t reads input frames t0+t .. t0+t+KT-1 (the
 * caller keeps the causal cache frames in front). mode 0: out bf16 [T_out][H][W][out_ld]
 * = acc + bias (+ resid[pix*resid_ld + n]); mode 1: time split, channel block j of
 * Cout/2 goes to output frame 2t+j; mode 2: uint8 RGB = clamp(rint((acc+bias+1)*127.5)).
 * Bits 8-10 of mode select the kernel of this call (0 auto; tests / A/B benchmarks): 1 per-tap
 * boxes, 2 dx reuse (one haloed TMA box per (dt,dy) feeds the 3 dx taps) on CTA pairs, 3 dx reuse
 * on single CTAs, 4 CTA pairs with one 128-pixel M-subtile per CTA (auto uses two at Cout 96). */
int ftb_conv3d_bf16(const void* in, int32_t T_in, int32_t H, int32_t W, int32_t Cin,
                    const void* w_t, int32_t Cout, int32_t KT, int32_t KH, int32_t KW, int32_t t0,
                    const float* bias, const void* resid, int64_t resid_ld,
                    void* out, int64_t out_ld, int32_t T_out, int32_t mode, void* stream);
/* Spatially split decode: as ftb_conv3d_bf16 (3x3 spatial kernels) but input rows -1 and H come
 * from halo_top / halo_bot, each [T_in][1][W][Cin] bf16 (the neighbour ranks' edge rows, or zeros
 * at the global edge) instead of zero padding. */
int ftb_conv3d_halo_bf16(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in, int32_t H,
                         int32_t W, int32_t Cin, const void* w_t, int32_t Cout, int32_t KT, int32_t KH, int32_t KW,
                         int32_t t0, const float* bias, const void* resid, int64_t resid_ld, void* out,
                         int64_t out_ld, int32_t T_out, int32_t mode, void* stream);
/* Fused RMS norm (+SiLU) of the conv output over all Cout channels (Wan RMS_norm:
 * y = x / max(||x||_2, 1e-12) * sqrt(C) * gamma), written as bf16 channel-last
 * [T_out][H][W][ld] — the next conv's input — in the same epilogue. */
typedef struct ftb_conv_norm {
  const float* gamma;  /* [Cout] */
  void* out;           /* bf16 */
  int64_t ld;
  int32_t silu;
  int32_t write_main;  /* 0: skip the main output (`out` of the conv may be NULL, no residual) */
} ftb_conv_norm;
/* As ftb_conv3d_halo_bf16 (halos may both be NULL) with the fused norm; store mode 0 and
 * Cout <= 192 (one N tile holds every channel of a pixel). */
int ftb_conv3d_norm_bf16(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in, int32_t H,
                         int32_t W, int32_t Cin, const void* w_t, int32_t Cout, int32_t KT, int32_t KH, int32_t KW,
                         int32_t t0, const float* bias, const void* resid, int64_t resid_ld, void* out,
                         int64_t out_ld, int32_t T_out, int32_t mode, const ftb_conv_norm* norm, void* stream);
/* RGB8 head of the decoder (3x3x3 causal conv, Cout = 3, uint8 RGB = clamp(rint((acc+bias+1)*127.5)))
 * as a 1x1 GEMM per input frame with the 27 taps x 3 channels as its 81 output rows,
 * Y[t][tap*3 + c][p] = sum_k w[c][k][tap] x[t][p][k] (w_taps bf16 [81][Cin], row tap*3 + c, tap =
 * (dt*3 + dy)*3 + dx), stored tap-major per frame in the caller's bf16 workspace (>= 81 *
 * (T_in*H*W + [2*T_in*W with halos]) elements), then a gather kernel summing each output pixel's
 * 27 shifted taps. Output frame t reads input frames t0+t .. t0+t+2; spatial zero padding or halo rows as
 * in ftb_conv3d_halo_bf16. out: uint8 [T_out][H][W][3]. */
int ftb_conv3d_head_rgb8(const void* in, const void* halo_top, const void* halo_bot, int32_t T_in, int32_t H,
                         int32_t W, int32_t Cin, const void* w_taps, const float* bias, void* y_ws,
                         int64_t y_ws_elems, void* out, int32_t T_out, int32_t t0, void* stream);
/* y = [silu](x / max(||x||_2, eps) * sqrt(C) * gamma) per pixel, channel-last bf16. */
int ftb_rmsnorm_silu_bf16(const void* x, int64_t n_pix, int32_t C, const float* gamma, float eps,
                          int32_t silu, void* y, void* stream);
/* Nearest 2x spatial upsample, channel-last bf16 [T][H][W][C] -> [T][2H][2W][C]. */
int ftb_upsample2x_bf16(const void* x, int32_t T, int32_t H, int32_t W, int32_t C, void* y, void* stream);
/* fp32 residual-stream variants: RMS norm (+SiLU) f32 -> bf16; nearest 2x upsample f32 -> bf16.
 * conv3d `mode` also carries flags: bit 4 = fp32 output, bit 5 = fp32 residual. */
int ftb_rmsnorm_silu_f32(const float* x, int64_t n_pix, int32_t C, const float* gamma, float eps, int32_t silu,
                         void* y, void* stream);
int ftb_upsample2x_f32_bf16(const float* x, int32_t T, int32_t H, int32_t W, int32_t C, void* y, void* stream);
/* Sampler latents f32 [T][C][H][W] -> channel-last bf16 [T][H][W][ldy]. */
int ftb_nchw_to_nhwc_bf16(const float* x, int32_t T, int32_t C, int32_t H, int32_t W, void* y, int32_t ldy,
                          void* stream);

/* Decoder mid-block attention (single head over a frame's H*W pixels, head_dim = C):
 * p[r][j] = bf16(softmax_j(s[r][j] * scale)) for fp32 scores s [rows][ld_s] (one CTA per row,
 * any cols), and a bf16 transpose y[c][r] = x[r][c] ([rows][ld_x] -> [cols][ld_y]) that turns V
 * into the K-major operand of the P.V GEMM. */
int ftb_softmax_rows_bf16(const float* s, int64_t ld_s, int32_t rows, int32_t cols, float scale, void* p,
                          int64_t ld_p, void* stream);
int ftb_transpose_bf16(const void* x, int64_t ld_x, int32_t rows, int32_t cols, void* y, int64_t ld_y,
                       void* stream);

/* Counter-based N(0,1)*scale fill (synthetic random-init weights at 14B shape). */
int ftb_fill_normal_bf16(void* out, int64_t n, uint64_t seed, float scale, void* stream);
int ftb_fill_normal_f32(float* out, int64_t n, uint64_t seed, float scale, void* stream);

/* Reduce: out[0] = count of non-finite values in x (f32), for NumericError checks. */
int ftb_count_nonfinite(const float* x, int64_t n, int32_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
