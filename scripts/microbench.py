"""Kernel microbenchmarks on the B200 vs library bars (cuBLAS matmul, torch SDPA).
Times with CUDA events over R repetitions after warm-up; inputs > L2 where it matters."""
import json
import math
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
    dev = torch.device("cuda")
    res = {}
    L = 10530
    for (M, N, K, tag) in [(L, 3 * 5120, 5120, "qkv14b"), (L, 5120, 5120, "o14b"), (L, 13824, 5120, "ffn1_14b"),
                           (L, 5120, 13824, "ffn2_14b"), (L, 4608, 1536, "qkv1.3b"), (8192, 8192, 8192, "sq8k")]:
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        w = torch.randn(N, K, device=dev).to(torch.bfloat16) / math.sqrt(K)
        out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        t = timeit(lambda: ops.gemm(a, w, out, "bf16"))
        tc = timeit(lambda: torch.matmul(a, w.t(), out=out))
        fl = 2.0 * M * N * K
        res[tag] = {"ours_ms": t, "ours_tflops": fl / t / 1e9, "cublas_ms": tc, "cublas_tflops": fl / tc / 1e9}
        print(tag, res[tag], flush=True)
    for (Lq, H, hd, tag) in [(L, 40, 128, "attn14b"), (L, 12, 128, "attn1.3b"), (L, 5, 128, "attn14b_sp8")]:
        q = torch.randn(Lq, H * hd, device=dev).to(torch.bfloat16)
        k = torch.randn(Lq, H * hd, device=dev).to(torch.bfloat16)
        v = torch.randn(Lq, H * hd, device=dev).to(torch.bfloat16)
        o = torch.empty_like(q)
        t = timeit(lambda: ops.attention(q, k, v, o, H, hd, Lq, Lq, 1 / math.sqrt(hd), impl=0), reps=5)
        qt, kt, vt = (x.view(Lq, H, hd).transpose(0, 1).unsqueeze(0) for x in (q, k, v))
        ts = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), reps=5)
        fl = 4.0 * Lq * Lq * H * hd
        res[tag] = {"ours_ms": t, "ours_tflops": fl / t / 1e9, "sdpa_ms": ts, "sdpa_tflops": fl / ts / 1e9}
        print(tag, res[tag], flush=True)
    json.dump(res, open("gpurun_out/microbench.json", "w"), indent=1)


if __name__ == "__main__":
    main()
