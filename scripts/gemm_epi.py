"""Epilogue cost at a short-K shape (the folded cross-attention output GEMM 10530x5120x1600)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402
from scripts.gemm_shapes import timeit  # noqa: E402

dev = torch.device("cuda")
L, N = 10530, 5120
for K in (1600, 5120):
    a = torch.randn(L, K, device=dev).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
    for kind in ("bf16", "f32", "resid_f32"):
        out = torch.zeros(L, N, device=dev, dtype=torch.float32 if kind.endswith("f32") else torch.bfloat16)
        t = timeit(lambda: ops.gemm(a, w, out, kind))
        print("K=%d %-10s %.3f ms %.0f TFLOP/s" % (K, kind, t, 2.0 * L * N * K / t / 1e9), flush=True)
