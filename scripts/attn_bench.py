"""FMHA variant check + timing: each impl vs torch SDPA on the 14B/1.3B shapes and
ragged cases. Usage: python scripts/attn_bench.py [impl ...]"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402


def timeit(fn, reps=5, warm=2):
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
    impls = [int(a) for a in sys.argv[1:]] or [0]
    dev = torch.device("cuda")
    torch.manual_seed(0)
    for (Lq, Lk, H, hd) in [(300, 300, 2, 128), (257, 70, 3, 64), (1000, 129, 2, 128), (4096, 4096, 4, 64),
                            (1000, 37, 4, 128), (777, 128, 2, 64), (2000, 16, 3, 128), (130, 1, 1, 128)]:
        q, k, v = (torch.randn(L, H * hd, device=dev).to(torch.bfloat16) for L in (Lq, Lk, Lk))
        qt, kt, vt = (x.view(-1, H, hd).transpose(0, 1).float() for x in (q, k, v))
        ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt).transpose(0, 1).reshape(Lq, H * hd)
        for impl in impls:
            if impl == 3 and Lk > 128:
                continue
            o = torch.zeros(Lq, H * hd, device=dev, dtype=torch.bfloat16)
            ops.attention(q, k, v, o, H, hd, Lq, Lk, 1 / math.sqrt(hd), impl=impl)
            torch.cuda.synchronize()
            err = ((o.float() - ref).norm() / ref.norm()).item()
            print("check impl=%d Lq=%d Lk=%d H=%d hd=%d rel=%.2e" % (impl, Lq, Lk, H, hd, err), flush=True)
    L = 10530
    q = torch.randn(L, 40 * 128, device=dev).to(torch.bfloat16)
    kv = torch.randn(37, 2 * 40 * 128, device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    for impl in impls:
        if impl in (0, 3):
            t = timeit(lambda: ops.attention(q, kv[:, :5120], kv[:, 5120:], o, 40, 128, L, 37, 0.088, impl=impl))
            print("cross14b impl=%d %.1f us  %.0f GB/s (Q read + O write)" % (impl, t * 1e3, 2 * q.numel() * 2 / t / 1e6),
                  flush=True)
    import statistics
    for (H, hd, tag) in [(40, 128, "attn14b"), (12, 128, "attn1.3b"), (5, 128, "attn14b_g8")]:
        q, k, v = (torch.randn(L, H * hd, device=dev).to(torch.bfloat16) for _ in range(3))
        o = torch.empty_like(q)
        ws = ops.attention_workspace(L, L, H, hd, dev)
        fl = 4.0 * L * L * H * hd
        qs, ks, vs = (x.view(1, L, H, hd).transpose(1, 2) for x in (q, k, v))
        runs = {}
        for _ in range(5):   # interleaved: same clocks / power state for every variant
            for impl in [i for i in impls if i != 3]:
                for w_, wn in ((None, ""), (ws, "+split")):
                    if w_ is None and ws is not None and impl == 0 and len(impls) > 1:
                        continue
                    t = timeit(lambda: ops.attention(q, k, v, o, H, hd, L, L, 1 / math.sqrt(hd), impl=impl,
                                                     workspace=w_))
                    runs.setdefault("impl=%d%s" % (impl, wn), []).append(t)
            t = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qs, ks, vs))
            runs.setdefault("torch_sdpa", []).append(t)
        for name, ts in runs.items():
            t = statistics.median(ts)
            print("%s %-16s %.3f ms %.0f TFLOP/s" % (tag, name, t, fl / t / 1e9), flush=True)


if __name__ == "__main__":
    main()
