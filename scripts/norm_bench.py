"""Norm + AdaLN at the 14B / 1.3B row shapes: time (CUDA events) and achieved GB/s.
usage: python scripts/norm_bench.py [--diag]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import ops  # noqa: E402
from scripts.gemm_shapes import timeit  # noqa: E402


def main():
    dev = torch.device("cuda")
    variants = [0]
    L = 10530
    for m in (5120, 1536):
        h = torch.randn(L, m, device=dev) * 3 + 0.5
        mod = torch.randn(10, 2 * m, device=dev)
        mod2 = torch.randn(91, 2 * m, device=dev)
        g = torch.randn(m, device=dev)
        b = torch.randn(m, device=dev)
        ref = None
        for var in variants:
            u = torch.empty(L, m, device=dev, dtype=torch.bfloat16)
            cases = [("adaln", dict(shift=mod[:, :m], scale=mod[:, m:], rows_per_group=1170)),
                     ("affine", dict(gamma=g, beta=b))]
            if "--diag" in sys.argv:
                cases += [("adaln1g", dict(shift=mod[:, :m], scale=mod[:, m:], rows_per_group=L)),
                          ("scale", dict(scale=mod[:, m:], rows_per_group=1170)),
                          ("shift", dict(shift=mod[:, :m], rows_per_group=1170)),
                          ("adaln_ld0", dict(shift=mod[:1, :m].expand(10, m), scale=mod[:1, m:].expand(10, m),
                                             rows_per_group=1170)),
                          ("adaln_g117", dict(shift=mod2[:, :m], scale=mod2[:, m:], rows_per_group=117)),
                          ("plain", dict()),
                          ("gamma", dict(gamma=g))]
            for tag, kw in cases:
                fn = lambda: ops.norm_modulate(h, u, **kw)  # noqa: E731
                t = timeit(fn, reps=50)
                byt = L * m * 6
                same = ""
                if tag == "adaln":
                    if ref is None:
                        ref = u.clone()
                    else:
                        same = "bit-equal" if torch.equal(ref, u) else "DIFF max %.3g" % (ref.float() - u.float()).abs().max()
                print("m=%d var=%d %-6s %.1f us %.0f GB/s %s" % (m, var, tag, t * 1e3, byt / t / 1e6, same), flush=True)


if __name__ == "__main__":
    main()
