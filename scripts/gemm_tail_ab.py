"""Interleaved A/B of two ftb_set_gemm_variant values on the residual GEMM shapes: every
repetition times both variants back to back (same clocks / power state), medians reported.
usage: python scripts/gemm_tail_ab.py [a=0] [b=32] [reps=15]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402


def timed(fn, n=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def main():
    va = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    vb = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    dev = torch.device("cuda")
    L = 10530
    for (N, K, tag) in [(1536, 1536, "o_1.3b"), (1536, 8960, "ffn2_1.3b"), (5120, 5120, "o_14b"),
                        (5120, 13824, "ffn2_14b"), (5120, 1600, "xpb_14b")]:
        a = torch.randn(L, K, device=dev).to(torch.bfloat16)
        w = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
        out = torch.zeros(L, N, device=dev)
        bias = torch.zeros(N, device=dev)
        gate = torch.randn(28, N, device=dev)
        fn = lambda: ops.gemm(a, w, out, "resid_f32", bias=bias, group_vec=gate, rows_per_group=(L + 27) // 28)
        res = {va: [], vb: []}
        for _ in range(3):
            fn()
        for _ in range(reps):
            for v in (va, vb):
                A.call("ftb_set_gemm_variant", v)
                fn()
                torch.cuda.synchronize()
                res[v].append(timed(fn))
        A.call("ftb_set_gemm_variant", 0)
        ma, mb = statistics.median(res[va]), statistics.median(res[vb])
        print("%-10s K=%-6d v%d %.4f ms  v%d %.4f ms  (%+.1f %%)" % (tag, K, va, ma, vb, mb, 100 * (mb / ma - 1)),
              flush=True)


if __name__ == "__main__":
    main()
