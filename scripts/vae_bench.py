"""Decode timing of the 14B-shape chunk (7 latents of 16x52x90 -> 28 RGB8 frames 416x720)
for the norm-fusion modes of DeviceVAEDecoder: python scripts/vae_bench.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig  # noqa: E402


def main():
    dev = torch.device("cuda")
    z = torch.randn(7, 16, 52, 90, device=dev)
    s = torch.cuda.current_stream()
    from paper_2512_23379_b200 import _capi as A
    variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
    for var, mode in [(v, "all") for v in variants] * 2:
        A.CONV_VARIANT = var   # conv mode bits 8-10 of every call (vae._conv)
        dec = DeviceVAEDecoder(VAEConfig(z_dim=16), dev, params=None, seed=201, rgb8=True, fuse_norm=mode)
        for _ in range(2):
            dec.decode_device_tensor(z, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            dec.decode_device_tensor(z, s)
        e1.record()
        torch.cuda.synchronize()
        print("conv variant %d fuse_norm=%-5s decode %.1f ms" % (var, mode, e0.elapsed_time(e1) / 5), flush=True)
        del dec
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
