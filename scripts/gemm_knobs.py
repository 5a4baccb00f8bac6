"""Time one GEMM shape under per-call kernel knobs (variant bits, raster group), interleaved:
python scripts/gemm_knobs.py M N K kind [variant,...] [group,...]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402


def main():
    M, N, K = (int(x) for x in sys.argv[1:4])
    kind = sys.argv[4]
    variants = [int(x) for x in sys.argv[5].split(",")] if len(sys.argv) > 5 else [0]
    groups = [int(x) for x in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0]
    dev = torch.device("cuda")
    a = (torch.randn(M, K, device=dev) / 4).to(torch.bfloat16)
    w = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
    out = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if kind in ("bf16", "gelu_bf16") else torch.float32)
    gate = torch.randn(10, N, device=dev)
    kw = dict(group_vec=gate, rows_per_group=1170) if kind == "resid_f32" else {}
    res = {}
    for _ in range(7):
        for v in variants:
            for g in groups:
                A.GEMM_GROUP = g
                fn = lambda: ops.gemm(a, w, out, kind, variant=v, **kw)  # noqa: E731
                for _ in range(2):
                    fn()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(5):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                res.setdefault((v, g), []).append(e0.elapsed_time(e1) / 5)
    for (v, g), ts in res.items():
        t = statistics.median(ts)
        print("%dx%dx%d %s variant=%d group=%d  %.1f us  %.0f TFLOP/s" % (M, N, K, kind, v, g, t * 1e3,
                                                                         2.0 * M * N * K / t / 1e9), flush=True)


if __name__ == "__main__":
    main()
