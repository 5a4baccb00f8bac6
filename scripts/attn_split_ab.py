"""Interleaved A/B of the flash kernel's KV-split tail round (ftb_set_attention_variant 0 = on,
1 = off) at the 14B (40 heads) and 1.3B (12 heads) self-attention shapes: medians of
back-to-back timings in one process. usage: python scripts/attn_split_ab.py [reps=15]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402


def timed(fn, n=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
    dev = torch.device("cuda")
    L, hd = 10530, 128
    for heads, tag in ((40, "14b"), (12, "1.3b")):
        m = heads * hd
        qkv = torch.randn(L, 3 * m, device=dev).to(torch.bfloat16)
        q, k, v = qkv[:, :m], qkv[:, m:2 * m], qkv[:, 2 * m:]
        o = torch.empty(L, m, device=dev, dtype=torch.bfloat16)
        fn = lambda: ops.attention(q, k, v, o, heads, hd, L, L, hd ** -0.5, impl=0)  # noqa: E731
        res = {0: [], 1: []}
        for v_ in (0, 1):
            A.call("ftb_set_attention_variant", v_)
            fn()
        torch.cuda.synchronize()
        for _ in range(reps):
            for v_ in (0, 1):
                A.call("ftb_set_attention_variant", v_)
                res[v_].append(timed(fn))
        A.call("ftb_set_attention_variant", 0)
        a, b = statistics.median(res[0]), statistics.median(res[1])
        fl = 4.0 * L * L * heads * hd
        print("%-5s split %.3f ms (%.0f TFLOP/s)  whole %.3f ms (%.0f TFLOP/s)  %+.1f %%"
              % (tag, a, fl / a / 1e9, b, fl / b / 1e9, 100 * (a / b - 1)), flush=True)


if __name__ == "__main__":
    main()
