"""RGB head formulations at the 14B decode shape (28 frames 416x720, 96 channels): the 1x1 GEMM
tap-major (M = 81 tap-channels, N = pixels) vs pixel-major (M = pixels, N = 96 / 112 / 128), and
the whole ftb_conv3d_head_rgb8. python scripts/head_bench.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200 import _capi as A  # noqa: E402
from paper_2512_23379_b200 import ops  # noqa: E402


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    dev = torch.device("cuda")
    T, H, W, C = 28, 416, 720, 96
    npix = (T + 2) * H * W
    x = torch.randn(npix, C, device=dev).to(torch.bfloat16)
    w = (torch.randn(128, C, device=dev) / 50).to(torch.bfloat16)
    b = torch.zeros(3, device=dev)
    ws = torch.empty(128 * npix, dtype=torch.bfloat16, device=dev)
    rgb = torch.empty(T * H * W * 3, dtype=torch.uint8, device=dev)
    full = t(lambda: A.call("ftb_conv3d_head_rgb8", A.ptr(x), None, None, T + 2, H, W, C, A.ptr(w), A.ptr(b),
                            A.ptr(ws), ws.numel(), A.ptr(rgb), T, 0, A.stream_ptr()))
    print("ftb_conv3d_head_rgb8 %.3f ms" % full)
    Y = ws[:81 * npix].view(81, npix)
    print("tap-major  M=81 N=pix   %.3f ms" % t(lambda: ops.gemm(w[:81], x, Y, "bf16")))
    fr = H * W
    Yf = ws[:81 * npix].view(T + 2, 81, fr)
    xf = x.view(T + 2, fr, C)

    def per_frame():
        for f in range(T + 2):
            ops.gemm(w[:81], xf[f], Yf[f], "bf16")
    print("tap-major per frame (30 x M=81 N=%d) %.3f ms" % (fr, t(per_frame)))
    for n in (96, 112, 128):
        Yp = ws[:npix * n].view(npix, n)
        print("pixel-major M=pix N=%d %.3f ms" % (n, t(lambda: ops.gemm(x, w[:n], Yp, "bf16"))))


if __name__ == "__main__":
    main()
