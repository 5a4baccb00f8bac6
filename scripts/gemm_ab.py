"""A/B of ftb_set_gemm_variant values on the residual-epilogue GEMM shapes.
usage: python scripts/gemm_ab.py 0,8,4 [tags]"""
import sys

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from scripts import gemm_shapes  # noqa: E402


def main():
    variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 8]
    tags = sys.argv[2] if len(sys.argv) > 2 else "xpb_14b,o_14b,ffn2_14b,xpb_1.3b,o_1.3b,ffn2_1.3b"
    for v in variants:
        print("variant", v, flush=True)
        A.call("ftb_set_gemm_variant", v)
        sys.argv = ["x", tags]
        gemm_shapes.main()
    A.call("ftb_set_gemm_variant", 0)


if __name__ == "__main__":
    main()
