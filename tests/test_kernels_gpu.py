"""Kernel-level numerics on the B200: every sm_100a kernel against a plain
PyTorch fp32 reference of the same op on the same (bf16-exact) inputs.

Tolerances: fp32-output GEMMs accumulate in fp32 over bf16 inputs that are
exactly representable, so they match an fp32 matmul to ~1e-5 relative;
bf16 outputs add one rounding (<= 2^-8 relative); attention stores P in bf16
(flash kernel) -> 1e-2 relative L2 (the north-star bf16 budget).
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).norm() / b.norm().clamp_min(1e-30))


def bf(x):
    return x.to(torch.bfloat16)


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2512_23379_b200 import ops as O
    return O


GEMM_SHAPES = [(128, 256, 64), (9, 32, 24), (9, 8, 32), (300, 200, 160), (1000, 768, 1536),
               (257, 64, 96), (2048, 1536, 1536), (130, 4608, 512), (64, 48, 200)]


@pytest.mark.parametrize("M,N,K", GEMM_SHAPES)
def test_gemm_f32_bias(ops, cuda, M, N, K):
    g = torch.Generator(device="cpu").manual_seed(M * 7 + N)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    out = torch.empty(M, N, device=cuda)
    ops.gemm(a, w, out, "f32", bias=b)
    ref = a.float() @ w.float().t() + b
    torch.cuda.synchronize()
    assert rel(out, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(300, 200, 160), (1024, 1024, 512)])
def test_gemm_bf16_and_gelu(ops, cuda, M, N, K):
    g = torch.Generator().manual_seed(3)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm(a, w, out, "bf16", bias=b)
    ref = a.float() @ w.float().t() + b
    assert rel(out.float(), ref) < 5e-3
    ops.gemm(a, w, out, "gelu_bf16", bias=b)
    refg = 0.5 * ref * (1 + torch.tanh(math.sqrt(2 / math.pi) * (ref + 0.044715 * ref ** 3)))
    assert rel(out.float(), refg) < 5e-3


def test_gemm_resid_gate_and_rowadd(ops, cuda):
    g = torch.Generator().manual_seed(5)
    M, N, K, rpg = 9 * 40, 256, 128, 40
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    gate = torch.randn(9, N, generator=g).to(cuda)
    h = torch.randn(M, N, generator=g).to(cuda)
    h0 = h.clone()
    ops.gemm(a, w, h, "resid_f32", bias=b, group_vec=gate, rows_per_group=rpg)
    grp = torch.arange(M, device=cuda) // rpg
    ref = h0 + gate[grp] * (a.float() @ w.float().t() + b)
    assert rel(h, ref) < 1e-5
    ops.gemm(a, w, h, "resid_f32")
    assert rel(h, ref + a.float() @ w.float().t()) < 1e-5
    out = torch.empty(M, N, device=cuda)
    ops.gemm(a, w, out, "rowadd_f32", bias=b, group_vec=gate, rows_per_group=rpg)
    assert rel(out, a.float() @ w.float().t() + b + gate[grp]) < 1e-5


@pytest.mark.parametrize("M,N,K", [(1000, 512, 1600), (300, 1536, 64), (10530 // 8, 5120, 256), (600, 1600, 320)])
def test_gemm_resid_staged_matches_row_per_thread(ops, cuda, M, N, K):
    """The smem-staged residual epilogue of the pair kernel is bit-identical to the
    row-per-thread one (ragged M, gate groups that straddle 32-row warp spans)."""
    g = torch.Generator().manual_seed(M + K)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    gate = torch.randn(7, N, generator=g).to(cuda)
    h0 = torch.randn(M, N, generator=g).to(cuda)
    outs = []
    for variant in (0, 6):  # staged vs row-per-thread (pair kernel), per-call selection
        h = h0.clone()
        ops.gemm(a, w, h, "resid_f32", bias=b, group_vec=gate, rows_per_group=(M + 6) // 7, variant=variant)
        outs.append(h)
    assert torch.equal(outs[0], outs[1])
    grp = torch.arange(M, device=cuda) // ((M + 6) // 7)
    assert rel(outs[0], h0 + gate[grp] * (a.float() @ w.float().t() + b)) < 1e-5
    # plain fp32 output (+ bias) through the same staged path, ragged last N tile included
    f32 = []
    for variant in (0, 6):
        o = torch.full((M, N), float("nan"), device=cuda)
        ops.gemm(a, w, o, "f32", bias=b, variant=variant)
        f32.append(o)
    assert torch.equal(f32[0], f32[1])
    assert rel(f32[0], a.float() @ w.float().t() + b) < 1e-5


@pytest.mark.parametrize("M,N,K", [(10530, 5120, 8192),   # 840 tiles: 26-tile tail in 2 K-slices
                                   (10530, 1536, 8960),   # 1.3B FFN2 shape: 252 tiles, 30 in 2 slices
                                   (47 * 256 - 100, 512, 8192),  # 94 tiles: 20 in 3 slices
                                   (46 * 256 - 7, 512, 8320)])   # 92 tiles: 18 in 4 slices
def test_gemm_resid_split_tail(ops, cuda, M, N, K):
    """Residual pair GEMM whose partial last wave runs as K-slices on the idle pairs: matches
    the fp32 reference, is deterministic launch to launch (the slices add into h in a fixed
    order, counters re-armed by each launch) and agrees with the unsplit kernel to rounding.
    The counters are the caller's (no library state); without them the tail runs unsplit."""
    g = torch.Generator().manual_seed(M + N + K)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    gate = torch.randn(28, N, generator=g).to(cuda)
    h0 = torch.randn(M, N, generator=g).to(cuda)
    rpg = (M + 27) // 28
    ctr = torch.zeros(ops.A.TAIL_COUNTER_WORDS, dtype=torch.int32, device=cuda)
    outs = []
    for split in (True, True, True, False):
        h = h0.clone()
        ops.gemm(a, w, h, "resid_f32", bias=b, group_vec=gate, rows_per_group=rpg,
                 tail_counters=ctr if split else None)
        outs.append(h)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert int(ctr.abs().sum()) == 0          # every launch leaves its counters re-armed
    grp = torch.arange(M, device=cuda) // rpg
    ref = h0 + gate[grp] * (a.float() @ w.float().t() + b)
    assert rel(outs[0], ref) < 1e-5
    assert rel(outs[0], outs[3]) < 5e-6
    # the tail tiles really were split: the last m-blocks differ from the unsplit result
    # only by fp32 rounding of the slice sums (not bit-identical)
    assert not torch.equal(outs[0], outs[3])


@pytest.mark.parametrize("M,N,K", [(37, 10240, 512), (1, 5120, 16), (100, 4096, 256)])
def test_gemm_few_rows(ops, cuda, M, N, K):
    """Few m-blocks: narrowed single-CTA tiles (grid spread over the SMs)."""
    g = torch.Generator().manual_seed(M * 7 + K)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm(a, w, out, "bf16")
    assert rel(out.float(), a.float() @ w.float().t()) < 5e-3


@pytest.mark.parametrize("M,heads,J,n_cond,K", [(700, 13, 40, 37, 256), (100, 40, 40, 37, 128), (300, 7, 48, 48, 64),
                                                 (513, 3, 8, 5, 512)])
def test_seg_softmax_epilogue(ops, cuda, M, heads, J, n_cond, K):
    """Logits GEMM with the per-head softmax in its epilogue == fp32 torch reference (logits,
    softmax over each head's first n_cond keys, padded keys exactly 0), pair kernel at M >= 256,
    single-CTA tiles below."""
    g = torch.Generator().manual_seed(M + J)
    u = bf(torch.randn(M, K, generator=g)).to(cuda)
    at = bf(torch.randn(heads * J, K, generator=g) / math.sqrt(K) * 4).to(cuda)
    s = (u.float() @ at.float().t()).reshape(M, heads, J)
    p_ref = torch.zeros(M, heads, J, device=cuda)
    p_ref[..., :n_cond] = torch.softmax(s[..., :n_cond], dim=-1)
    p_ref = p_ref.reshape(M, heads * J)
    spt = 256 // J
    at_t = torch.zeros((heads + spt - 1) // spt * 256, K, device=cuda, dtype=torch.bfloat16)
    at_t[ops.tiled_seg_rows(heads, J).to(cuda)] = at
    p = torch.full((M, heads * J), float("nan"), device=cuda, dtype=torch.bfloat16)
    ops.xattn_logits_softmax(u, at_t, p, heads, J, n_cond)
    assert rel(p.float(), p_ref) < 4e-3
    assert float((p.float() - p_ref).abs().max()) < 4e-3
    pad = p.float().reshape(M, heads, J)[..., n_cond:]
    assert pad.numel() == 0 or int((pad != 0).sum()) == 0


def test_gemm_chunked_a(ops, cuda):
    """Ulysses gather layout: A's K dim arrives as g head-group slices."""
    g = torch.Generator().manual_seed(9)
    chunks, M, kc, N = 4, 300, 128, 192
    raw = bf(torch.randn(chunks, M, kc, generator=g)).to(cuda)
    w = bf(torch.randn(N, chunks * kc, generator=g) / 20).to(cuda)
    out = torch.empty(M, N, device=cuda)
    ops.gemm(raw, w, out, "f32", M=M, K=chunks * kc, lda=kc, a_chunks=chunks, a_chunk_stride=M * kc)
    a = raw.permute(1, 0, 2).reshape(M, chunks * kc)
    assert rel(out, a.float() @ w.float().t()) < 1e-5


def _rope_tables(frames, gh, gw, hd, theta=10000.0):
    from paper_2512_23379_b200.rope import rope3d_tables
    return rope3d_tables(frames, gh, gw, hd, theta)


@pytest.mark.parametrize("hpr", [4, 2, 1])
def test_gemm_qkv_rope_layout(ops, cuda, hpr):
    from paper_2512_23379_b200.ops import RopeTables
    heads, hd, frames, gh, gw = 4, 64, 3, 4, 6
    m = heads * hd
    M = frames * gh * gw
    g = torch.Generator().manual_seed(2)
    a = bf(torch.randn(M, m, generator=g)).to(cuda)
    w = bf(torch.randn(3 * m, m, generator=g) / 16).to(cuda)
    tabs = _rope_tables(frames, gh, gw, hd)
    rt = RopeTables(tabs, gh, gw, cuda)
    out = torch.empty(M * 3 * m, device=cuda, dtype=torch.bfloat16)
    ops.gemm(a, w, out.view(M, 3 * m), "qkv_rope", heads=heads, head_dim=hd, heads_per_rank=hpr, rope=rt)
    y = (a.float() @ w.float().t()).cpu().double().numpy().reshape(M, 3, heads, hd)
    # reference rotation on (q, k)
    ang = np.zeros((M, hd // 2))
    pt, ph, pw = tabs["cos_t"].shape[1], tabs["cos_h"].shape[1], tabs["cos_w"].shape[1]
    cos = np.zeros((M, hd // 2))
    sin = np.zeros((M, hd // 2))
    for t in range(M):
        f, rem = divmod(t, gh * gw)
        yy, xx = divmod(rem, gw)
        cos[t] = np.concatenate([tabs["cos_t"][f], tabs["cos_h"][yy], tabs["cos_w"][xx]])
        sin[t] = np.concatenate([tabs["sin_t"][f], tabs["sin_h"][yy], tabs["sin_w"][xx]])
    ref = y.copy()
    for which in (0, 1):
        x0, x1 = y[:, which, :, 0::2], y[:, which, :, 1::2]
        ref[:, which, :, 0::2] = x0 * cos[:, None] - x1 * sin[:, None]
        ref[:, which, :, 1::2] = x0 * sin[:, None] + x1 * cos[:, None]
    g_ = heads // hpr
    got = out.float().cpu().double().numpy().reshape(g_, M, 3, hpr, hd)
    got = got.transpose(1, 2, 0, 3, 4).reshape(M, 3, heads, hd)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 5e-3
    del ang, pt, ph, pw


def torch_attn(q, k, v, heads, hd, scale):
    Lq, Lk = q.shape[0], k.shape[0]
    qh = q.float().view(Lq, heads, hd).transpose(0, 1)
    kh = k.float().view(Lk, heads, hd).transpose(0, 1)
    vh = v.float().view(Lk, heads, hd).transpose(0, 1)
    p = torch.softmax(qh @ kh.transpose(1, 2) * scale, dim=-1)
    return (p @ vh).transpose(0, 1).reshape(Lq, heads * hd)


@pytest.mark.parametrize("Lq,Lk,heads,hd", [(128, 128, 1, 128), (300, 300, 2, 128), (1170, 1170, 3, 128),
                                            (500, 777, 2, 64), (2340, 2340, 2, 128), (129, 1000, 1, 64)])
def test_fmha_tcgen05(ops, cuda, Lq, Lk, heads, hd):
    g = torch.Generator().manual_seed(Lq + Lk)
    q = bf(torch.randn(Lq, heads * hd, generator=g)).to(cuda)
    k = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    v = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    o = torch.empty(Lq, heads * hd, device=cuda, dtype=torch.bfloat16)
    scale = 1 / math.sqrt(hd)
    ops.attention(q, k, v, o, heads, hd, Lq, Lk, scale, impl=0)
    assert rel(o.float(), torch_attn(q, k, v, heads, hd, scale)) < 1e-2


def test_fmha_strided_qkv_layout(ops, cuda):
    """q|k|v interleaved per token ([L, 3, H, hd]) as produced by the QKV epilogue."""
    L, heads, hd = 700, 3, 128
    g = torch.Generator().manual_seed(1)
    qkv = bf(torch.randn(L, 3 * heads * hd, generator=g) * 2).to(cuda)
    m = heads * hd
    q, k, v = qkv[:, :m], qkv[:, m:2 * m], qkv[:, 2 * m:]
    o = torch.empty(L, m, device=cuda, dtype=torch.bfloat16)
    ops.attention(q, k, v, o, heads, hd, L, L, 1 / math.sqrt(hd), impl=0)
    assert rel(o.float(), torch_attn(q, k, v, heads, hd, 1 / math.sqrt(hd))) < 1e-2


@pytest.mark.parametrize("Lq,Lk,heads,hd", [(1170, 37, 4, 128), (10530 // 8, 37, 5, 128), (300, 128, 2, 64),
                                            (129, 1, 1, 128), (2000, 65, 3, 128), (64, 16, 2, 64)])
def test_xattn_short_kv(ops, cuda, Lq, Lk, heads, hd):
    """Short-KV tcgen05 kernel (cross-attention, Lk <= 128): TMA-stored output into a
    strided view (only its own head columns written) and the default dispatch."""
    g = torch.Generator().manual_seed(Lq + 7 * Lk)
    q = bf(torch.randn(Lq, heads * hd, generator=g) * 2).to(cuda)
    kv = bf(torch.randn(Lk, 2 * heads * hd, generator=g)).to(cuda)
    k, v = kv[:, :heads * hd], kv[:, heads * hd:]
    big = torch.full((Lq, heads * hd + 64), 7.0, device=cuda).to(torch.bfloat16)
    o = big[:, :heads * hd]
    scale = 1 / math.sqrt(hd)
    ops.attention(q, k, v, o, heads, hd, Lq, Lk, scale, impl=3)
    want = torch_attn(q, k, v, heads, hd, scale)
    assert rel(o.float(), want) < 5e-3
    assert torch.all(big[:, heads * hd:] == 7.0)          # TMA store clipped to the view
    o2 = torch.empty_like(o)
    ops.attention(q, k, v, o2, heads, hd, Lq, Lk, scale)  # default dispatch picks the same kernel
    assert torch.equal(o2, o)


def test_xattn_scatter_rows(ops, cuda):
    """Ulysses scatter epilogue on the short-KV kernel: row r -> peer r // rows."""
    Lq, Lk, heads, hd, g_ = 300, 37, 2, 128, 3
    gen = torch.Generator().manual_seed(3)
    q = bf(torch.randn(Lq, heads * hd, generator=gen)).to(cuda)
    k = bf(torch.randn(Lk, heads * hd, generator=gen)).to(cuda)
    v = bf(torch.randn(Lk, heads * hd, generator=gen)).to(cuda)
    rows = Lq // g_
    outs = [torch.zeros(rows, heads * hd, device=cuda, dtype=torch.bfloat16) for _ in range(g_)]
    ops.attention_scatter(q, k, v, heads, hd, Lq, Lk, 0.1, [t.data_ptr() for t in outs], rows, heads * hd)
    want = torch_attn(q, k, v, heads, hd, 0.1)
    assert rel(torch.cat(outs).float(), want) < 5e-3


@pytest.mark.parametrize("Lq,Lk,heads,hd", [(9, 9, 2, 16), (9, 10, 2, 16), (1170, 37, 4, 128), (100, 70, 3, 64),
                                            (5, 3, 4, 8), (33, 100, 2, 32)])
def test_attention_small(ops, cuda, Lq, Lk, heads, hd):
    g = torch.Generator().manual_seed(Lq * 3 + Lk)
    q = bf(torch.randn(Lq, heads * hd, generator=g)).to(cuda)
    k = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    v = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    o = torch.empty(Lq, heads * hd, device=cuda, dtype=torch.bfloat16)
    scale = 1 / math.sqrt(hd)
    ops.attention(q, k, v, o, heads, hd, Lq, Lk, scale, impl=1)
    assert rel(o.float(), torch_attn(q, k, v, heads, hd, scale)) < 5e-3


@pytest.mark.parametrize("M,N", [(9, 32), (300, 1536), (17, 5120), (5, 6144), (7, 1000), (3, 1030), (4, 8200)])
def test_norm_modulate(ops, cuda, M, N):
    g = torch.Generator().manual_seed(N)
    x = (torch.randn(M, N, generator=g) * 3 + 1.5).to(cuda)
    gam, bet = torch.randn(N, generator=g).to(cuda), torch.randn(N, generator=g).to(cuda)
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    mean = torch.empty(M, device=cuda)
    rstd = torch.empty(M, device=cuda)
    ops.norm_modulate(x, out, gamma=gam, beta=bet, mean_out=mean, rstd_out=rstd)
    mu = x.double().mean(1)
    var = x.double().var(1, unbiased=False)
    rs = 1 / torch.sqrt(var + 1e-6)
    ref = (x.double() - mu[:, None]) * rs[:, None] * gam.double() + bet.double()
    assert rel(out.float(), ref.float()) < 5e-3
    assert rel(mean, mu.float()) < 1e-5 and rel(rstd, rs.float()) < 1e-5
    # AdaLN: per-group (1 + scale), shift
    G = 3
    rpg = (M + G - 1) // G
    mod = torch.randn(G, 2, N, generator=g).to(cuda)
    ops.norm_modulate(x, out, scale=mod[:, 0], shift=mod[:, 1], rows_per_group=rpg)
    grp = torch.arange(M, device=cuda) // rpg
    ref2 = (x.double() - mu[:, None]) * rs[:, None] * (1 + mod[grp, 0].double()) + mod[grp, 1].double()
    assert rel(out.float(), ref2.float()) < 5e-3


def test_patchify_unpatch_roundtrip(ops, cuda):
    Lm, Lc, D, H, W, ph, pw = 2, 5, 3, 4, 6, 2, 2
    g = torch.Generator().manual_seed(0)
    motion = torch.randn(Lm, D, H, W, generator=g)
    z = torch.randn(Lc - Lm, D, H, W, generator=g)
    ref = torch.randn(D, H, W, generator=g)
    F = (2 * D + 1) * ph * pw
    ldo = 32
    T = (H // ph) * (W // pw)
    out = torch.empty(Lc * T, ldo, dtype=torch.bfloat16, device=cuda)
    ops.patchify(motion.to(cuda), z.to(cuda), ref.to(cuda), Lm, Lc, D, H, W, ph, pw, out)
    # numpy reference of Eq.1 + patchify
    zn = torch.cat([motion, z]).numpy()
    mask = np.zeros((Lc, 1, H, W))
    mask[0] = 1
    cond = np.zeros((Lc, D, H, W))
    cond[0] = ref.numpy()
    st = np.concatenate([zn, mask, cond], axis=1)  # (Lc, C, H, W)
    C_ = st.shape[1]
    tok = st.reshape(Lc, C_, H // ph, ph, W // pw, pw).transpose(0, 2, 4, 1, 3, 5).reshape(Lc * T, C_ * ph * pw)
    got = out.float().cpu().numpy()
    assert np.allclose(got[:, :F], tok.astype(np.float32), atol=2e-2, rtol=1e-2)
    assert np.all(got[:, F:] == 0)
    # unpatch: x0 tokens -> frames, with DDIM update
    x0t = torch.randn(Lc * T, 16, generator=g).to(cuda)
    zs = torch.randn(Lc - Lm, D, H, W, generator=g).to(cuda)
    z0 = zs.clone()
    x0o = torch.empty(Lc - Lm, D, H, W, device=cuda)
    ops.unpatch_ddim(x0t[:, :D * ph * pw], Lm, Lc, D, H, W, ph, pw, zs, x0o, coeffs=(0.25, 0.75, 0.5, 0.5))
    xt = x0t[:, :D * ph * pw].cpu().numpy().reshape(Lc, H // ph, W // pw, D, ph, pw)
    frames = xt.transpose(0, 3, 1, 4, 2, 5).reshape(Lc, D, H, W)[Lm:]
    assert np.allclose(x0o.cpu().numpy(), frames, atol=1e-6)
    eps = (z0.cpu().numpy() - 0.25 * frames) / 0.75
    assert np.allclose(zs.cpu().numpy(), 0.5 * frames + 0.5 * eps, atol=1e-5)


def test_fill_normal_statistics(ops, cuda):
    t = torch.empty(1 << 22, device=cuda, dtype=torch.bfloat16)
    ops.fill_normal_(t, 1234, 1.0)
    x = t.float()
    assert abs(float(x.mean())) < 5e-3 and abs(float(x.std()) - 1) < 5e-3
    t2 = torch.empty_like(t)
    ops.fill_normal_(t2, 1234, 1.0)
    assert torch.equal(t, t2)


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (300, 512, 160), (1000, 768, 1536), (2048, 1536, 1536),
                                   (10530 // 4, 1024, 512), (257, 4608, 96)])
def test_gemm_variants(ops, cuda, variant, M, N, K):
    """Single-CTA and CTA-pair (cta_group::2) kernels give the same fp32 result."""
    g = torch.Generator().manual_seed(M + N + K)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    b = torch.randn(N, generator=g).to(cuda)
    h = torch.randn(M, N, generator=g).to(cuda)
    h0 = h.clone()
    out = torch.empty(M, N, device=cuda)
    ops.gemm(a, w, out, "f32", bias=b, variant=variant)
    ops.gemm(a, w, h, "resid_f32", bias=b, variant=variant)
    ob = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm(a, w, ob, "gelu_bf16", bias=b, variant=variant)
    ref = a.float() @ w.float().t() + b
    assert rel(out, ref) < 1e-5
    assert rel(h, h0 + ref) < 1e-5
    refg = 0.5 * ref * (1 + torch.tanh(math.sqrt(2 / math.pi) * (ref + 0.044715 * ref ** 3)))
    assert rel(ob.float(), refg) < 5e-3


@pytest.mark.parametrize("heads,hd,n_cond", [(40, 128, 37), (12, 128, 37), (7, 64, 9)])
def test_gemm_block_diagonal_band(ops, cuda, heads, hd, n_cond):
    """Fold GEMMs over the block-diagonal K / V operands with the K-band skip (each pair tile's
    K loop covers only its rows' head bands) == the dense K loop bit for bit (the skipped
    products are exact zeros), and == an fp32 reference of the block-diagonal product."""
    m, J = heads * hd, (n_cond + 7) // 8 * 8
    spt = 256 // J
    g = torch.Generator().manual_seed(heads * hd)
    kv = bf(torch.randn(n_cond, 2 * m, generator=g)).to(cuda)
    wq = bf(torch.randn(m, m, generator=g) / math.sqrt(m)).to(cuda)
    wo = bf(torch.randn(m, m, generator=g) / math.sqrt(m)).to(cuda)
    at_rows = (heads + spt - 1) // spt * 256
    kbd = torch.zeros(at_rows, m, dtype=torch.bfloat16, device=cuda)
    vbd = torch.zeros(heads * J, m, dtype=torch.bfloat16, device=cuda)
    ops.xattn_blockdiag(kv, kbd, vbd, n_cond, heads, hd, J, 0.125, k_tiled=True)
    res = []
    for band in (False, True):
        at = torch.full((at_rows, m), float("nan"), dtype=torch.bfloat16, device=cuda)
        bt = torch.full((m, heads * J), float("nan"), dtype=torch.bfloat16, device=cuda)
        ops.gemm(kbd, wq, at, "bf16", band=(0, J, 256, spt, hd) if band else None)
        ops.gemm(wo, vbd, bt, "bf16", band=(1, J, 0, 0, hd) if band else None)
        res.append((at, bt))
    torch.cuda.synchronize()
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert rel(res[1][0].float(), kbd.float() @ wq.float().t()) < 5e-3
    assert rel(res[1][1].float(), wo.float() @ vbd.float().t()) < 5e-3


def test_gemm_resid_split_tail_graph_replay(ops, cuda):
    """The split-K tail's slice counters (caller-owned) are re-armed by every launch, so a
    captured launch replays to the same bits as eager launches sharing the same counters."""
    M, N, K = 10530, 5120, 8192
    g = torch.Generator().manual_seed(11)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / math.sqrt(K)).to(cuda)
    gate = torch.randn(28, N, generator=g).to(cuda)
    h0 = torch.randn(M, N, generator=g).to(cuda)
    rpg = (M + 27) // 28
    ctr = torch.zeros(ops.A.TAIL_COUNTER_WORDS, dtype=torch.int32, device=cuda)
    h = h0.clone()
    ops.gemm(a, w, h, "resid_f32", group_vec=gate, rows_per_group=rpg, tail_counters=ctr)
    eager = h.clone()
    s = torch.cuda.Stream(device=cuda)
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    hg = h0.clone()
    with torch.cuda.stream(s):
        ops.gemm(a, w, hg, "resid_f32", group_vec=gate, rows_per_group=rpg, stream=s, tail_counters=ctr)  # warm-up
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            ops.gemm(a, w, hg, "resid_f32", group_vec=gate, rows_per_group=rpg, stream=s, tail_counters=ctr)
    for _ in range(3):
        hg.copy_(h0)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(hg, eager)


@pytest.mark.parametrize("Lq,Lk,heads,hd", [(4000, 4000, 10, 128), (4000, 3000, 10, 64), (10530, 10530, 12, 128)])
def test_fmha_kv_split_tail(ops, cuda, Lq, Lk, heads, hd):
    """Flash attention whose partial last round of (head, 256-query) items runs as two key
    halves per item plus a combine kernel: every head matches the fp32 reference, the whole
    items are bit-identical to the unsplit launch, and the split items differ from it only by
    rounding (so the split really ran). The workspace is the caller's."""
    sms = torch.cuda.get_device_properties(cuda).multi_processor_count
    n_qblk = (Lq + 255) // 256
    items, R = n_qblk * heads, (n_qblk * heads) % sms
    assert items > sms and 0 < 2 * R <= sms  # the shapes are chosen to take the split path
    g = torch.Generator().manual_seed(Lq + Lk + hd)
    q = bf(torch.randn(Lq, heads * hd, generator=g) * 2).to(cuda)
    k = bf(torch.randn(Lk, heads * hd, generator=g) * 2).to(cuda)
    v = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    scale = 1 / math.sqrt(hd)
    ws = ops.attention_workspace(Lq, Lk, heads, hd, cuda)
    assert ws is not None and ws.numel() * 4 == ops.attention_workspace_bytes(Lq, Lk, heads, hd) > 0
    outs = []
    for w_ in (ws, None):
        o = torch.full((Lq, heads * hd), float("nan"), device=cuda, dtype=torch.bfloat16)
        ops.attention(q, k, v, o, heads, hd, Lq, Lk, scale, impl=0, workspace=w_)
        outs.append(o)
    torch.cuda.synchronize()
    split, whole = outs
    first = items - R                      # first split item: head first // n_qblk
    h0 = first // n_qblk
    for h in sorted({0, h0, heads - 1}):
        cols = slice(h * hd, (h + 1) * hd)
        want = torch_attn(q[:, cols], k[:, cols], v[:, cols], 1, hd, scale)
        assert rel(split[:, cols].float(), want) < 1e-2, h
    r0 = (first % n_qblk) * 256
    assert torch.equal(split[:, :h0 * hd], whole[:, :h0 * hd])
    assert torch.equal(split[:r0, h0 * hd:(h0 + 1) * hd], whole[:r0, h0 * hd:(h0 + 1) * hd])
    tail = (split[:, (heads - 1) * hd:].float() - whole[:, (heads - 1) * hd:].float())
    assert 0 < float(tail.norm() / whole[:, (heads - 1) * hd:].float().norm()) < 5e-3


def test_fmha_kv_split_graph_replay(ops, cuda):
    """KV-split attention captured in a CUDA graph on a capture stream and replayed on another
    stream: the workspace is the caller's (not keyed by stream handle), so replays reproduce the
    eager bits, also with a second workspace-owning launch of another shape interleaved."""
    Lq = Lk = 10530
    heads, hd = 12, 128
    g = torch.Generator().manual_seed(21)
    q = bf(torch.randn(Lq, heads * hd, generator=g) * 2).to(cuda)
    k = bf(torch.randn(Lk, heads * hd, generator=g) * 2).to(cuda)
    v = bf(torch.randn(Lk, heads * hd, generator=g)).to(cuda)
    ws = ops.attention_workspace(Lq, Lk, heads, hd, cuda)
    assert ws is not None
    eager = torch.empty(Lq, heads * hd, device=cuda, dtype=torch.bfloat16)
    ops.attention(q, k, v, eager, heads, hd, Lq, Lk, 0.088, impl=0, workspace=ws)
    cap = torch.cuda.Stream(device=cuda)
    cap.wait_stream(torch.cuda.current_stream())
    o = torch.empty_like(eager)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        ops.attention(q, k, v, o, heads, hd, Lq, Lk, 0.088, impl=0, workspace=ws, stream=cap)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cap):
            ops.attention(q, k, v, o, heads, hd, Lq, Lk, 0.088, impl=0, workspace=ws, stream=cap)
    other = torch.cuda.Stream(device=cuda)
    q2 = bf(torch.randn(4000, 10 * 128, generator=g)).to(cuda)
    ws2 = ops.attention_workspace(4000, 4000, 10, 128, cuda)
    o2 = torch.empty_like(q2)
    for _ in range(3):
        o.zero_()
        with torch.cuda.stream(other):
            graph.replay()
            ops.attention(q2, q2, q2, o2, 10, 128, 4000, 4000, 0.088, impl=0, workspace=ws2, stream=other)
        torch.cuda.synchronize()
        assert torch.equal(o, eager)


@pytest.mark.parametrize("rows,cols", [(1, 1), (37, 5), (300, 4680), (9, 1031)])
def test_softmax_rows_and_transpose(ops, cuda, rows, cols):
    """The decoder mid attention's helpers: fp32 row softmax -> bf16 P (vs torch fp32, bf16
    rounding), and the bf16 transpose (bit-exact), on ragged shapes with padded leading dims."""
    g = torch.Generator().manual_seed(rows * 7 + cols)
    ldp = (cols + 7) // 8 * 8 + 8
    s = torch.empty(rows, ldp, device=cuda)[:, :cols]
    s.copy_((torch.randn(rows, cols, generator=g) * 4).to(cuda))
    p = torch.full((rows, ldp), 7.0, device=cuda, dtype=torch.bfloat16)
    ops.softmax_rows_bf16(s, p[:, :cols], 0.3)
    ref = torch.softmax(s * 0.3, dim=-1)
    assert torch.allclose(p[:, :cols].float(), ref, atol=1e-3, rtol=8e-3)
    assert torch.all(p[:, cols:] == 7.0)          # nothing written past the row
    x = bf(torch.randn(rows, cols, generator=g)).to(cuda)
    y = torch.full((cols, rows + 8), -1.0, device=cuda, dtype=torch.bfloat16)
    ops.transpose_bf16(x, y[:, :rows])
    assert torch.equal(y[:, :rows], x.t())
    assert torch.all(y[:, rows:] == -1.0)


@pytest.mark.parametrize("M,N,K", [(10530, 1536, 480), (300, 1536, 1536), (257, 2592, 544), (1000, 5120, 1024)])
def test_gemm_resid_tma_staged_epilogue(ops, cuda, M, N, K):
    """Short-K fp32 residual GEMMs take the TMA-staged h epilogue (whole h boxes in and out by
    TMA): bit-identical to the per-thread staged epilogue (variant bit 32), within fp32
    rounding of an fp32 reference, and nothing written outside the logical rows / columns."""
    g = torch.Generator().manual_seed(M + N + K)
    a = bf(torch.randn(M, K, generator=g)).to(cuda)
    w = bf(torch.randn(N, K, generator=g) / K ** 0.5).to(cuda)
    gate = torch.randn(10, N, generator=g).to(cuda)
    bias = torch.randn(N, generator=g).to(cuda)
    pad = 8
    base = torch.randn(M + 64, N + pad, generator=g).to(cuda)
    outs = []
    for var in (0, 32):
        buf = base.clone()
        ops.gemm(a, w, buf[:M, :N], "resid_f32", group_vec=gate, rows_per_group=1170, bias=bias, variant=var)
        outs.append(buf)
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0][:, N:], base[:, N:]) and torch.equal(outs[0][M:], base[M:])
    ref = base[:M, :N] + gate.repeat_interleave(1170, 0)[:M] * (a.float() @ w.float().t() + bias)
    assert ((outs[0][:M, :N] - ref).norm() / (ref - base[:M, :N]).norm()).item() < 1e-5
