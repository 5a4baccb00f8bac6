"""Raster-group sweep (ftb_set_gemm_group) on chosen GEMM shapes.
usage: python scripts/gemm_group.py 0,4,8,15,21,42 [tags]"""
import sys

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from scripts import gemm_shapes  # noqa: E402


def main():
    groups = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 8, 15, 42]
    tags = sys.argv[2] if len(sys.argv) > 2 else "o_14b,ffn2_14b,qkv_14b,ffn1_14b,xpb_14b"
    for g in groups:
        print("group", g, flush=True)
        A.call("ftb_set_gemm_group", g)
        sys.argv = ["x", tags]
        gemm_shapes.main()
    A.call("ftb_set_gemm_group", 0)


if __name__ == "__main__":
    main()
