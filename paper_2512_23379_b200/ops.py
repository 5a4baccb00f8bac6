"""Device-tensor wrappers over the C-ABI kernels (torch tensors for memory and
streams only; all arithmetic happens in libftb2.so).

Conventions: activations are row-major with an explicit leading dimension
(row stride); weights are stored transposed, W^T [N, K] bf16 (K-major), which
is the tcgen05 B-operand layout. The reference stores (in, out) and computes
x @ W + b (`backends/reference.py:17-18`); W^T is the same matrix.
"""

import contextlib
import ctypes as C
import os

import torch

from . import _capi as A
from .errors import ConfigError

# Optional per-launch profiler (bench.py roofline pass): list of
# (kind, start_event, end_event, flops, bytes) or None.
PROFILER = None
PROFILE_DETAIL = None  # set to True: per-shape GEMM buckets


class _Prof:
    def __init__(self, kind, flops, nbytes, stream):
        self.on = PROFILER is not None
        if self.on:
            self.kind, self.flops, self.nbytes = kind, flops, nbytes
            self.s = stream if stream is not None else torch.cuda.current_stream()
            self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        if self.on:
            self.e0.record(self.s)
        return self

    def __exit__(self, *exc):
        if self.on:
            self.e1.record(self.s)
            PROFILER.append((self.kind, self.e0, self.e1, self.flops, self.nbytes))
        return False


_NVTX = os.environ.get("FTB_NVTX", "1") != "0"


def nvtx_push(name):
    if _NVTX and torch.cuda.is_available():
        torch.cuda.nvtx.range_push(name)


def nvtx_pop():
    if _NVTX and torch.cuda.is_available():
        torch.cuda.nvtx.range_pop()


@contextlib.contextmanager
def nvtx(name):
    """NVTX range around a stage (chunk, ladder step, DiT layer, decode) for nsys / ncu
    --nvtx filtering; host-side markers only (inside a captured graph they mark the capture)."""
    on = _NVTX and torch.cuda.is_available()
    if on:
        torch.cuda.nvtx.range_push(name)
    try:
        yield
    finally:
        if on:
            torch.cuda.nvtx.range_pop()


KINDS = {"bf16": A.EPI_BF16, "gelu_bf16": A.EPI_GELU_BF16, "f32": A.EPI_F32,
         "resid_f32": A.EPI_RESID_F32, "rowadd_f32": A.EPI_ROWADD_F32, "qkv_rope": A.EPI_QKV_ROPE,
         "seg_softmax": A.EPI_SEG_SOFTMAX}


def _ld(t):
    if t.dim() != 2 or t.stride(1) != 1:
        raise ConfigError("expected a 2-d row-major tensor (unit column stride)")
    return t.stride(0)


def _need(t, dtype, name):
    if not t.is_cuda or t.dtype != dtype:
        raise ConfigError("%s must be a CUDA %s tensor" % (name, dtype))


class RopeTables:
    """Device copy of the host-computed 3D RoPE tables (rope.py), expanded per
    token: cos/sin [frames*grid_h*grid_w][head_dim/2] float32."""

    def __init__(self, tables, grid_h, grid_w, device):
        from .rope import per_token_tables
        cos, sin = per_token_tables(tables, grid_h, grid_w)
        self.cos = torch.as_tensor(cos).contiguous().to(device)
        self.sin = torch.as_tensor(sin).contiguous().to(device)
        self.struct = A.Rope3D(A.ptr(self.cos), A.ptr(self.sin))


def gemm(a, w_t, out, kind="bf16", *, bias=None, group_vec=None, rows_per_group=0, row_offset=0,
         M=None, K=None, lda=None, a_chunks=1, a_chunk_stride=0, heads=0, head_dim=0,
         heads_per_rank=0, rope=None, peers=None, band=None, stream=None, algo_flops=None, variant=None,
         tail_counters=None, prof_kind=None):
    """out <- epilogue(a[M,K] @ w_t[N,K]^T). `a` may be a raw buffer when
    a_chunks > 1 (Ulysses gather: M, K, lda, a_chunk_stride explicit).
    peers: device addresses (ints) for the peer-store epilogues (qkv_rope: one
    receive block per head group; f32: replicated all-gather); `out` then only
    fixes dtype/ldc.
    band: (side, rows, tile, per_tile, k) — the A (side 0) or B (side 1) operand is block
    diagonal (ftb_epilogue.band_*); tiles skip the K blocks outside their rows' bands.
    variant: kernel selection of this call (ftb_epilogue.variant; None = FTB_GEMM_VARIANT or 0).
    tail_counters: caller-owned int32 [TAIL_COUNTER_WORDS] zeroed buffer enabling the split-K
    tail wave of long-K residual GEMMs (one buffer per stream of launches)."""
    _need(a, torch.bfloat16, "A")
    _need(w_t, torch.bfloat16, "W^T")
    N, Kw = w_t.shape
    if M is None:
        M, K = a.shape
        lda = _ld(a)
    if K > Kw or (K != Kw and (Kw - K) >= 8):
        raise ConfigError("gemm: K mismatch %d vs %d" % (K, Kw))
    k = KINDS[kind]
    ldc = 0 if k == A.EPI_QKV_ROPE else _ld(out)
    if k in (A.EPI_BF16, A.EPI_GELU_BF16, A.EPI_QKV_ROPE, A.EPI_SEG_SOFTMAX):
        _need(out, torch.bfloat16, "out")
    else:
        _need(out, torch.float32, "out")
    group_ld = 0
    if group_vec is not None:
        _need(group_vec, torch.float32, "group_vec")
        group_ld = _ld(group_vec)
    if bias is not None:
        _need(bias, torch.float32, "bias")
    epi = A.Epilogue(k, rows_per_group, row_offset, A.ptr(bias), A.ptr(group_vec), group_ld, A.ptr(out), ldc,
                     heads, head_dim, heads_per_rank, C.pointer(rope.struct) if rope is not None else None)
    if band is not None:
        epi.band_side, epi.band_rows, epi.band_tile, epi.band_per_tile, epi.band_k = (int(x) for x in band)
    epi.variant = A.GEMM_VARIANT if variant is None else int(variant)
    epi.raster_group = A.GEMM_GROUP
    if tail_counters is not None:
        if tail_counters.dtype != torch.int32 or tail_counters.numel() < A.TAIL_COUNTER_WORDS:
            raise ConfigError("tail_counters must be int32 with >= %d words" % A.TAIL_COUNTER_WORDS)
        epi.tail_counters = tail_counters.data_ptr()
    if peers:
        if len(peers) > A.MAX_PEERS:
            raise ConfigError("at most %d peers" % A.MAX_PEERS)
        epi.n_peers = len(peers)
        for i, pp in enumerate(peers):
            epi.peer_out[i] = int(pp)
    # algo_flops: the algorithmic FLOPs when the operands are structurally sparse (the
    # block-diagonal fold GEMMs), so the profile's TFLOP/s do not count multiplications by zero
    fl = 2.0 * M * N * K if algo_flops is None else float(algo_flops)
    pk = prof_kind or ("gemm" if PROFILE_DETAIL is None else "gemm:%s:%dx%dx%d" % (kind, M, N, K))
    with _Prof(pk, fl, 2.0 * (M * K + N * K) + out.element_size() * M * N, stream):
        A.call("ftb_gemm_bf16", A.ptr(a), lda, a_chunks, a_chunk_stride, A.ptr(w_t), _ld(w_t), M, N, K,
               C.byref(epi), A.stream_ptr(stream))
    return out


def norm_modulate(x, out, *, gamma=None, beta=None, scale=None, shift=None, rows_per_group=0, row_offset=0,
                  eps=1e-6, mean_out=None, rstd_out=None, stream=None):
    _need(x, torch.float32, "x")
    _need(out, torch.bfloat16, "out")
    M, N = x.shape
    mod_ld = 0
    for t in (scale, shift):
        if t is not None:
            mod_ld = _ld(t)
    if scale is not None and shift is not None and scale.stride(0) != shift.stride(0):
        raise ConfigError("scale/shift strides differ")
    with _Prof("norm", 0.0, 6.0 * M * N, stream):
        A.call("ftb_norm_modulate", A.ptr(x), _ld(x), M, N, A.ptr(gamma), A.ptr(beta), A.ptr(scale), A.ptr(shift),
               mod_ld, rows_per_group, row_offset, float(eps), A.ptr(out), _ld(out), A.ptr(mean_out),
               A.ptr(rstd_out), A.stream_ptr(stream))
    return out


def attention_probs(q, k, heads, head_dim, Lq, Lk, scale, out=None, stream=None):
    """softmax(q . k^T * scale) per head as fp32 [heads, Lq, Lk] (ftb_attention_probs): the p of
    the reference mha_forward cache (backends/reference.py:86-88), which the flash kernels
    never materialise."""
    _need(q, torch.bfloat16, "q")
    _need(k, torch.bfloat16, "k")
    if out is None:
        out = torch.empty(heads, Lq, Lk, dtype=torch.float32, device=q.device)
    _need(out, torch.float32, "out")
    A.call("ftb_attention_probs", A.ptr(q), _ld(q), A.ptr(k), _ld(k), int(Lq), int(Lk), int(heads), int(head_dim),
           float(scale), A.ptr(out), A.stream_ptr(stream))
    return out


def attention_workspace_bytes(Lq, Lk, heads, head_dim):
    """fp32 workspace bytes of the flash kernel's KV-split tail round for this shape (0: none)."""
    return int(A.lib.ftb_attention_workspace_bytes(int(Lq), int(Lk), int(heads), int(head_dim)))


def attention_workspace(Lq, Lk, heads, head_dim, device):
    """Caller-owned KV-split workspace (None when the shape has no split round or
    FTB_ATTN_NO_SPLIT=1); pass it to every attention call of that shape on one stream."""
    nb = attention_workspace_bytes(Lq, Lk, heads, head_dim) if A.ATTN_SPLIT else 0
    return torch.empty(nb // 4, dtype=torch.float32, device=device) if nb else None


def _ws(workspace):
    if workspace is None:
        return None, 0
    _need(workspace, torch.float32, "workspace")
    return A.ptr(workspace), workspace.numel() * 4


def attention(q, k, v, out, heads, head_dim, Lq, Lk, scale, *, impl=None, workspace=None, stream=None):
    """q/k/v/out are 2-d views (rows, ld) whose head h lives at columns
    [h*head_dim, (h+1)*head_dim). workspace: attention_workspace() of this shape (optional)."""
    for t, nm in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
        _need(t, torch.bfloat16, nm)
    args = (A.ptr(q), _ld(q), A.ptr(k), _ld(k), A.ptr(v), _ld(v), A.ptr(out), _ld(out),
            Lq, Lk, heads, head_dim, float(scale), *_ws(workspace), A.stream_ptr(stream))
    if impl is None:   # the library's dispatch (ftb_attention): short-KV tcgen05 kernel when Lk <= 128
        impl = (3 if Lk <= 128 else 0) if (head_dim in (64, 128) and Lq >= 64) else 1
    kind = {0: "fmha", 3: "xattn"}.get(impl, "attn_small")
    with _Prof(kind, 4.0 * Lq * Lk * heads * head_dim, 2.0 * heads * head_dim * (2 * Lq + 2 * Lk), stream):
        A.call("ftb_attention_impl", int(impl), *args)
    if impl == 0 and workspace is not None:
        A.LAUNCHES[0] += 1   # + fmha2_combine_kernel of the KV-split tail round
    return out


def attention_scatter(q, k, v, heads, head_dim, Lq, Lk, scale, o_peers, peer_rows, ldo, *, workspace=None,
                      stream=None):
    """attention() whose output row r lands in row r % peer_rows of the buffer at
    device address o_peers[r // peer_rows] (Ulysses all-to-all #2 in the epilogue)."""
    for t, nm in ((q, "q"), (k, "k"), (v, "v")):
        _need(t, torch.bfloat16, nm)
    if not (1 <= len(o_peers) <= A.MAX_PEERS):
        raise ConfigError("attention_scatter: 1..%d peers" % A.MAX_PEERS)
    arr = (C.c_void_p * len(o_peers))(*[int(x) for x in o_peers])
    kind = "fmha" if Lk > 128 else "xattn"
    with _Prof(kind, 4.0 * Lq * Lk * heads * head_dim, 2.0 * heads * head_dim * (2 * Lq + 2 * Lk), stream):
        A.call("ftb_attention_scatter", A.ptr(q), _ld(q), A.ptr(k), _ld(k), A.ptr(v), _ld(v), arr, len(o_peers),
               int(peer_rows), int(ldo), Lq, Lk, heads, head_dim, float(scale), *_ws(workspace),
               A.stream_ptr(stream))
    if Lk > 128 and workspace is not None:
        A.LAUNCHES[0] += 1   # + fmha2_combine_kernel


def peer_barrier(flag_ptrs, epoch, rank, world, timeout_s=30.0, *, stream=None):
    """Stream-ordered cross-rank barrier over peer-mapped flag words (dist.PeerComm)."""
    arr = (C.c_void_p * len(flag_ptrs))(*[int(x) for x in flag_ptrs])
    A.call("ftb_peer_barrier", arr, A.ptr(epoch), rank, world, float(timeout_s), A.stream_ptr(stream))


def patchify(motion, z, reference, Lm, Lc, D, H, W, ph, pw, out, stream=None):
    A.call("ftb_patchify_composite", A.ptr(motion) if Lm > 0 else None, A.ptr(z), A.ptr(reference),
           Lm, Lc, D, H, W, ph, pw, A.ptr(out), _ld(out), A.stream_ptr(stream))
    return out


def patchify_stacked(stacked, ph, pw, out, stream=None):
    """stacked f32 device [Lc][C][H][W] -> bf16 patch tokens (any composite)."""
    Lc, Cc, H, W = stacked.shape
    A.call("ftb_patchify_stacked", A.ptr(stacked), Lc, Cc, H, W, ph, pw, A.ptr(out), _ld(out), A.stream_ptr(stream))
    return out


def unpatch_ddim(x0_tok, Lm, Lc, D, H, W, ph, pw, z, x0_out, coeffs=None, stream=None):
    if coeffs is None:
        a_i = s_i = a_n = s_n = 0.0
        upd = 0
    else:
        a_i, s_i, a_n, s_n = coeffs
        upd = 1
    A.call("ftb_unpatch_ddim", A.ptr(x0_tok), _ld(x0_tok), Lm, Lc, D, H, W, ph, pw, A.ptr(z), A.ptr(x0_out),
           float(a_i), float(s_i), float(a_n), float(s_n), upd, A.stream_ptr(stream))


def codec_decode(latents, Q, out, stream=None):
    n, D = latents.shape
    A.call("ftb_codec_decode", A.ptr(latents), A.ptr(Q), A.ptr(out), n, D, A.stream_ptr(stream))
    return out


def silu_to_bf16(x, out, stream=None):
    A.call("ftb_silu_f32_to_bf16", A.ptr(x), A.ptr(out), x.numel(), A.stream_ptr(stream))
    return out


def cast_f32_bf16(x, out, stream=None):
    A.call("ftb_cast_f32_bf16", A.ptr(x), A.ptr(out), x.numel(), A.stream_ptr(stream))
    return out


def softmax_rows_bf16(s, out, scale, stream=None):
    """out[r] = bf16(softmax(s[r] * scale)) over 2-d views (fp32 scores, bf16 probabilities)."""
    _need(s, torch.float32, "s")
    _need(out, torch.bfloat16, "out")
    rows, cols = s.shape
    with _Prof("vae_attn", 0.0, float(rows) * cols * 6, stream):
        A.call("ftb_softmax_rows_bf16", A.ptr(s), _ld(s), rows, cols, float(scale), A.ptr(out), _ld(out),
               A.stream_ptr(stream))
    return out


def transpose_bf16(x, out, stream=None):
    """out[c][r] = x[r][c] over 2-d bf16 views."""
    _need(x, torch.bfloat16, "x")
    _need(out, torch.bfloat16, "out")
    rows, cols = x.shape
    A.call("ftb_transpose_bf16", A.ptr(x), _ld(x), rows, cols, A.ptr(out), _ld(out), A.stream_ptr(stream))
    return out


def gelu_bf16(x, out, stream=None):
    A.call("ftb_gelu_bf16", A.ptr(x), A.ptr(out), x.numel(), A.stream_ptr(stream))
    return out


def fill_normal_(t, seed, scale=1.0, stream=None):
    if t.dtype == torch.bfloat16:
        A.call("ftb_fill_normal_bf16", A.ptr(t), t.numel(), int(seed) & ((1 << 64) - 1), float(scale),
               A.stream_ptr(stream))
    elif t.dtype == torch.float32:
        A.call("ftb_fill_normal_f32", A.ptr(t), t.numel(), int(seed) & ((1 << 64) - 1), float(scale),
               A.stream_ptr(stream))
    else:
        raise ConfigError("fill_normal_: bf16 or f32 only")
    return t


def count_nonfinite(x, flag, stream=None):
    A.call("ftb_count_nonfinite", A.ptr(x), x.numel(), A.ptr(flag), A.stream_ptr(stream))
    return flag


def add_bcast(a, b, out, stream=None):
    """out[l, f, :] = a[f, :] + b[l, :]"""
    F, n = a.shape
    Lb = b.shape[0]
    A.call("ftb_add_bcast_f32", A.ptr(a), F, n, A.ptr(b), Lb, A.ptr(out), A.stream_ptr(stream))
    return out


def xattn_blockdiag(kv, kbd, vbd, n_cond, heads, head_dim, J, scale, *, k_tiled=False, stream=None):
    """Diagonal blocks of the tensor-core fold operands (elementwise.cu): kbd[(h,j)][h*hd+d] =
    scale * K[j][h*hd+d], vbd likewise from V; the rest of kbd / vbd must already be zero.
    k_tiled: kbd rows in the SEG_SOFTMAX tile order (tiled_seg_rows)."""
    for t, nm in ((kv, "kv"), (kbd, "kbd"), (vbd, "vbd")):
        _need(t, torch.bfloat16, nm)
    spt = 256 // J if k_tiled else 0
    need_k = (heads + spt - 1) // spt * 256 if k_tiled else heads * J
    if kbd.shape[1] != vbd.shape[1] or kbd.stride(0) != vbd.stride(0) or kbd.shape[0] < need_k or \
            vbd.shape[0] < heads * J:
        raise ConfigError("xattn_blockdiag: kbd / vbd must be [rows][m] with one row stride")
    A.call("ftb_xattn_blockdiag", A.ptr(kv), _ld(kv), n_cond, heads, head_dim, J, float(scale), A.ptr(kbd),
           A.ptr(vbd), _ld(kbd), spt, A.stream_ptr(stream))


def xattn_logits_softmax(u, at_tiled, p, heads, J, n_cond, *, M=None, stream=None):
    """Folded cross-attention logits with the per-head softmax fused into the GEMM epilogue:
    p[r][h*J + j] = softmax_j<n_cond((u . at^T)[r][h*J + j]). at_tiled holds the rows of at in
    the epilogue's tile layout (tiled_seg_rows): 256 // J heads per 256-row tile, padded."""
    spt = 256 // J
    n_pad = (heads + spt - 1) // spt * 256
    if at_tiled.shape[0] != n_pad:
        raise ConfigError("xattn_logits_softmax: at_tiled must have %d rows" % n_pad)
    return gemm(u, at_tiled, p, "seg_softmax", heads=heads, head_dim=J, heads_per_rank=n_cond, M=M,
                K=at_tiled.shape[1] if M is not None else None, lda=u.stride(0) if M is not None else None,
                stream=stream, algo_flops=2.0 * (u.shape[0] if M is None else M) * heads * J * at_tiled.shape[1])


def tiled_seg_rows(heads, J):
    """Row of the padded tile layout for each (head, j): head h -> tile h // (256 // J), slot
    h % (256 // J), row tile * 256 + slot * J + j (the SEG_SOFTMAX epilogue's column order)."""
    spt = 256 // J
    h = torch.arange(heads).repeat_interleave(J)
    j = torch.arange(J).repeat(heads)
    return (h // spt) * 256 + (h % spt) * J + j
