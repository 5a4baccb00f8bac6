"""Out-of-bounds write checks of our own (compute-sanitizer is closed on this GPU pool): every
kernel family writes its output into a window of a larger buffer whose guard bands (before,
after, and the row padding beyond the logical width) hold a sentinel; ragged shapes exercise
the partial tiles. Any store outside the logical output changes a guard."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu
GUARD = 4096


def guarded(shape, dtype, dev, pad_cols=8):
    """(buffer, view): view = rows x cols with row stride cols + pad_cols inside buffer, GUARD
    elements of sentinel before and after."""
    rows, cols = shape
    ld = cols + pad_cols
    buf = torch.empty(GUARD + rows * ld + GUARD, dtype=dtype, device=dev)
    sentinel = -12345.0 if dtype != torch.uint8 else 77
    buf.fill_(sentinel)
    view = buf[GUARD:GUARD + rows * ld].view(rows, ld)[:, :cols]
    return buf, view, ld, sentinel


def check(buf, ld, shape, sentinel):
    rows, cols = shape
    body = buf[GUARD:GUARD + rows * ld].view(rows, ld)
    assert torch.all(buf[:GUARD] == sentinel), "write before the output"
    assert torch.all(buf[GUARD + rows * ld:] == sentinel), "write after the output"
    assert torch.all(body[:, cols:] == sentinel), "write into the row padding"


@pytest.fixture(scope="module")
def ops(cuda):
    from paper_2512_23379_b200 import ops as O
    return O


def bf(*shape, scale=1.0, dev="cuda"):
    return (torch.randn(*shape, device=dev) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(300, 520, 256), (100, 192, 136), (257, 4616, 96), (1, 64, 16)])
@pytest.mark.parametrize("kind", ["f32", "bf16", "gelu_bf16", "resid_f32"])
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_gemm_stays_in_bounds(ops, cuda, M, N, K, kind, variant):
    if variant == 2 and (M < 256 or N < 256):
        pytest.skip("CTA pair needs M, N >= 256")
    dt = torch.bfloat16 if kind in ("bf16", "gelu_bf16") else torch.float32
    buf, out, ld, s = guarded((M, N), dt, cuda)
    if kind == "resid_f32":
        out.zero_()
    ops.gemm(bf(M, K), bf(N, K, scale=0.05), out, kind, bias=torch.randn(N, device=cuda), variant=variant)
    torch.cuda.synchronize()
    check(buf, ld, (M, N), s)
    assert torch.isfinite(out.float()).all()


@pytest.mark.parametrize("Lq,Lk,H,hd,impl", [(700, 700, 3, 128, 0), (300, 260, 2, 64, 0), (500, 37, 4, 128, 3),
                                             (9, 10, 2, 16, 1), (130, 1, 1, 128, 0)])
def test_attention_stays_in_bounds(ops, cuda, Lq, Lk, H, hd, impl):
    q, k, v = bf(Lq, H * hd), bf(Lk, H * hd), bf(Lk, H * hd)
    buf, out, ld, s = guarded((Lq, H * hd), torch.bfloat16, cuda)
    ops.attention(q, k, v, out, H, hd, Lq, Lk, 1 / math.sqrt(hd), impl=impl)
    torch.cuda.synchronize()
    check(buf, ld, (Lq, H * hd), s)


def test_attention_kv_split_stays_in_bounds(ops, cuda):
    Lq, H, hd = 2600, 222, 64       # 2442 items: 74 split into key halves + combine
    q = bf(Lq, H * hd)
    ws = ops.attention_workspace(Lq, Lq, H, hd, cuda)
    assert ws is not None
    wbuf = torch.full((GUARD + ws.numel() + GUARD,), -7.0, device=cuda)
    wview = wbuf[GUARD:GUARD + ws.numel()]
    buf, out, ld, s = guarded((Lq, H * hd), torch.bfloat16, cuda)
    ops.attention(q, q, q, out, H, hd, Lq, Lq, 0.125, impl=0, workspace=wview)
    torch.cuda.synchronize()
    check(buf, ld, (Lq, H * hd), s)
    assert torch.all(wbuf[:GUARD] == -7.0) and torch.all(wbuf[GUARD + ws.numel():] == -7.0)


@pytest.mark.parametrize("M,N", [(300, 1536), (37, 5120), (5, 512)])
def test_norm_stays_in_bounds(ops, cuda, M, N):
    buf, out, ld, s = guarded((M, N), torch.bfloat16, cuda)
    ops.norm_modulate(torch.randn(M, N, device=cuda), out, scale=torch.randn(3, N, device=cuda),
                      shift=torch.randn(3, N, device=cuda), rows_per_group=(M + 2) // 3)
    torch.cuda.synchronize()
    check(buf, ld, (M, N), s)


@pytest.mark.parametrize("T,H,W,Cin,Cout,k", [(2, 3, 130, 96, 96, (3, 3, 3)), (2, 3, 70, 64, 192, (3, 3, 3)),
                                              (3, 5, 9, 32, 96, (3, 3, 3)), (2, 4, 33, 128, 64, (1, 1, 1))])
def test_conv_stays_in_bounds(cuda, T, H, W, Cin, Cout, k):
    from paper_2512_23379_b200 import _capi as A
    kt = k[0]
    x = bf(T + kt - 1, H, W, Cin)
    wt = bf(Cout, k[0] * k[1] * k[2] * Cin, scale=0.05)
    buf, out, ld, s = guarded((T * H * W, Cout), torch.bfloat16, cuda)
    A.call("ftb_conv3d_bf16", A.ptr(x), T + kt - 1, H, W, Cin, A.ptr(wt), Cout, *k, 0, None, None, 0, A.ptr(out), ld,
           T, 0, A.stream_ptr())
    torch.cuda.synchronize()
    check(buf, ld, (T * H * W, Cout), s)
