"""Decode stage codecs.

`Codec` mirrors the reference's orthogonal per-frame codec
(`pkg/src/ftlk/world.py:181-210`): encode = x @ Q^T, decode = z @ Q, with the
decode of each chunk's target latents done on device (ftb_codec_decode) and
copied to pinned host memory. The wan-mode causal VAE decoder lives in
`vae.py` and exposes the same `decode_device` / `frames_per_latent` surface.
"""

import numpy as np
import torch

from . import ops
from .errors import ConfigError


class Codec:
    frames_per_latent = 1

    def __init__(self, Q):
        Q = np.asarray(Q, dtype=np.float64)
        if Q.ndim != 2 or Q.shape[0] != Q.shape[1]:
            raise ConfigError("codec matrix must be square")
        if np.max(np.abs(Q.T @ Q - np.eye(Q.shape[0]))) > 1e-9:
            raise ConfigError("codec matrix must be orthogonal")
        self.Q = Q
        self._dev = {}
        self._pinned = {}

    @classmethod
    def identity(cls, dim):
        return cls(np.eye(dim))

    def encode(self, frames):
        frames = np.asarray(frames, dtype=np.float64)
        if frames.shape[-1] != self.Q.shape[0]:
            raise ConfigError("frame dimension does not match codec")
        return frames @ self.Q.T

    def decode(self, latents):
        latents = np.asarray(latents, dtype=np.float64)
        if latents.shape[-1] != self.Q.shape[0]:
            raise ConfigError("latent dimension does not match codec")
        return latents @ self.Q

    def _bufs(self, lat, slot=0):
        D = self.Q.shape[0]
        n, dev = lat.shape[0], lat.device
        Qd = self._dev.get(dev)
        if Qd is None:
            Qd = torch.as_tensor(self.Q, dtype=torch.float32).to(dev)
            self._dev[dev] = Qd
        key = (dev, n, slot)
        bufs = self._pinned.get(key)
        if bufs is None:
            bufs = (torch.empty(n, D, dtype=torch.float32, device=dev),
                    torch.empty(n, D, dtype=torch.float32).pin_memory())
            self._pinned[key] = bufs
        return Qd, bufs

    def decode_device_tensor(self, latents_dev, stream=None, gather=False, slot=0):
        """latents_dev: device fp32 (n, D[,1,1]) -> device fp32 frames (n, D) (replicated decode:
        the codec is per frame, so `gather` has nothing to collect)."""
        lat = latents_dev.reshape(-1, self.Q.shape[0])
        Qd, (out, _) = self._bufs(lat, slot)
        ops.codec_decode(lat, Qd, out, stream=stream)
        return out

    def decode_device_async(self, latents_dev, stream, slot=0, gather=False):
        """Decode + D2H into pinned buffer `slot`, enqueued on `stream`: (host tensor, event)."""
        lat = latents_dev.reshape(-1, self.Q.shape[0])
        _, (out, host) = self._bufs(lat, slot)
        self.decode_device_tensor(latents_dev, stream, slot=slot)
        with torch.cuda.stream(stream):
            host.copy_(out, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return host, ev

    def decode_device(self, latents_dev, stream):
        """latents_dev: device fp32 (n, D[,1,1]) -> host float64 frames (n, D)."""
        host, ev = self.decode_device_async(latents_dev, stream)
        ev.synchronize()
        return host.numpy().astype(np.float64)
