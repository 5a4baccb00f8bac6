"""Run each hot kernel at its 14B-shape size a few times (for ncu capture).
usage: python scripts/profile_kernels.py [gemm|oproj|ffn2|xpb|xs|norm|fmha|cross|conv|all]"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402
from paper_2512_23379_b200 import _capi as A  # noqa: E402


def main(which):
    dev = torch.device("cuda")
    L, m, H, hd = 10530, 5120, 40, 128
    if which in ("gemm", "all"):
        a = torch.randn(L, m, device=dev).to(torch.bfloat16)
        w = (torch.randn(3 * m, m, device=dev) / 70).to(torch.bfloat16)
        out = torch.empty(L, 3 * m, device=dev, dtype=torch.bfloat16)
        groups = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
        for g in groups:
            A.GEMM_GROUP = g   # raster group of these calls (ftb_epilogue.raster_group)
            for _ in range(3):
                ops.gemm(a, w, out, "bf16")
    if which in ("oproj", "ffn2", "xpb", "all"):
        K = {"ffn2": 13824, "xpb": 1600}.get(which, m)   # xpb: folded cross-attention output GEMM
        a = torch.randn(L, K, device=dev).to(torch.bfloat16)
        w = (torch.randn(m, K, device=dev) / 70).to(torch.bfloat16)
        h = torch.randn(L, m, device=dev)
        gate = torch.randn(10, m, device=dev)
        for _ in range(3):
            ops.gemm(a, w, h, "resid_f32", group_vec=gate, rows_per_group=1170)
    if which in ("xs", "all"):   # folded cross-attn logits GEMM with the per-head softmax epilogue
        u = torch.randn(L, m, device=dev).to(torch.bfloat16)
        at = (torch.randn(7 * 256, m, device=dev) / 70).to(torch.bfloat16)
        pbuf = torch.empty(L, 40 * 40, device=dev, dtype=torch.bfloat16)
        for _ in range(3):
            ops.xattn_logits_softmax(u, at, pbuf, 40, 40, 37)
    if which in ("norm", "all"):
        h = torch.randn(L, m, device=dev)
        u = torch.empty(L, m, device=dev, dtype=torch.bfloat16)
        mod = torch.randn(10, 2 * m, device=dev)
        for _ in range(3):
            ops.norm_modulate(h, u, shift=mod[:, :m], scale=mod[:, m:], rows_per_group=1170)
    if which in ("fmha", "all"):
        q = torch.randn(L, H * hd, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        for _ in range(3):
            ops.attention(q, q, q, o, H, hd, L, L, 1 / math.sqrt(hd), impl=0)
    if which in ("cross", "all"):
        q = torch.randn(L, H * hd, device=dev).to(torch.bfloat16)
        kv = torch.randn(37, 2 * H * hd, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        for _ in range(3):
            ops.attention(q, kv[:, :H * hd], kv[:, H * hd:], o, H, hd, L, 37, 1 / math.sqrt(hd))
    if which in ("conv", "all"):
        T, Hh, W, C = 28, 416, 720, 96
        x = torch.randn((T + 2) * Hh * W * C, device=dev).to(torch.bfloat16)
        wt = (torch.randn(C, 27 * C, device=dev) / 50).to(torch.bfloat16)
        out = torch.empty(T * Hh * W * C, device=dev, dtype=torch.float32)
        for _ in range(3):
            A.call("ftb_conv3d_bf16", A.ptr(x), T + 2, Hh, W, C, A.ptr(wt), C, 3, 3, 3, 0, None, None, 0, A.ptr(out),
                   C, T, 16, A.stream_ptr())
    if which in ("convres", "all"):   # conv2 of a 96-ch resblock: fp32 residual in, fp32 x + normalised bf16 out
        import ctypes as Cty
        T, Hh, W, C = 28, 416, 720, 96
        x = torch.randn((T + 2) * Hh * W * C, device=dev).to(torch.bfloat16)
        wt = (torch.randn(C, 27 * C, device=dev) / 50).to(torch.bfloat16)
        res = torch.randn(T * Hh * W * C, device=dev)
        out = torch.empty(T * Hh * W * C, device=dev, dtype=torch.float32)
        nout = torch.empty(T * Hh * W * C, device=dev, dtype=torch.bfloat16)
        g = torch.ones(C, device=dev)
        b = torch.zeros(C, device=dev)
        nrm = A.ConvNorm(A.ptr(g), A.ptr(nout), C, 1, 1)
        for _ in range(3):
            A.call("ftb_conv3d_norm_bf16", A.ptr(x), None, None, T + 2, Hh, W, C, A.ptr(wt), C, 3, 3, 3, 0, A.ptr(b),
                   A.ptr(res), C, A.ptr(out), C, T, 16 | 32, Cty.byref(nrm), A.stream_ptr())
    torch.cuda.synchronize()
    print("ok", which)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
