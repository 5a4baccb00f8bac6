"""GEMM shapes of the 14B and 1.3B DiT with their epilogues (ours vs cuBLAS where comparable)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
    dev = torch.device("cuda")
    L = 10530
    for (N, K, kind, tag) in [(8960, 1536, "gelu_bf16", "ffn1_1.3b"), (1536, 1536, "resid_f32", "o_1.3b"),
                              (4608, 1536, "bf16", "qkv_1.3b"), (1536, 8960, "resid_f32", "ffn2_1.3b"),
                              (13824, 5120, "gelu_bf16", "ffn1_14b"), (5120, 5120, "resid_f32", "o_14b"),
                              (15360, 5120, "bf16", "qkv_14b"), (5120, 13824, "resid_f32", "ffn2_14b"),
                              (480, 1536, "f32", "xs_1.3b"), (1536, 480, "resid_f32", "xpb_1.3b"),
                              (1600, 5120, "f32", "xs_14b"), (5120, 1600, "resid_f32", "xpb_14b")]:
        if only and tag not in only:
            continue
        a = torch.randn(L, K, device=dev).to(torch.bfloat16)
        w = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
        out = torch.zeros(L, N, device=dev, dtype=torch.float32 if kind.endswith("f32") else torch.bfloat16)
        bias = torch.zeros(N, device=dev)
        t = timeit(lambda: ops.gemm(a, w, out, kind, bias=bias))
        print("%-10s %-10s %.3f ms %.0f TFLOP/s" % (tag, kind, t, 2.0 * L * N * K / t / 1e9), flush=True)


if __name__ == "__main__":
    main()
