"""CPU oracle (TEST INFRASTRUCTURE ONLY): float64 NumPy restatement of the
wan-mode streaming causal VAE decoder (paper_2512_23379_b200/vae.py).

Parity status: UNPINNED by the reference — the reference decodes with an
orthogonal per-frame codec (`pkg/src/ftlk/world.py:181-210`, pinned in
ftlk_oracle.codec_decode); the convolutional Wan-2.1-shaped decoder is the
builder-defined stand-in for the paper's VAE documented in
DESIGN.md. This restatement is written independently of the device code:
dense loops over taps, channel-last float64, explicit causal caches.
"""

import numpy as np


def dims_of(base, mult):
    return [base * mult[-1]] + [base * u for u in reversed(mult)]


def conv3d(x, w, b):
    """x [T_in, H, W, Cin]; w (Cout, Cin, kt, kh, kw); stride 1, spatial zero pad k//2,
    no time pad (caller supplies causal frames). Returns [T_in-kt+1, H, W, Cout].
    Direct sum over the taps, one float64 BLAS product (pixels, Cin) x (Cin, Cout) per tap."""
    cout, cin, kt, kh, kw = w.shape
    T_in, H, W, _ = x.shape
    ph, pw = kh // 2, kw // 2
    xp = np.zeros((T_in, H + 2 * ph, W + 2 * pw, cin))
    xp[:, ph:ph + H, pw:pw + W] = x
    T = T_in - kt + 1
    out = np.zeros((T, H, W, cout))
    for dt in range(kt):
        for dy in range(kh):
            for dx in range(kw):
                tap = xp[dt:dt + T, dy:dy + H, dx:dx + W].reshape(-1, cin)
                out += (tap @ w[:, :, dt, dy, dx].T).reshape(out.shape)
    return out + b


def rms(x, g, silu=True):
    n = np.sqrt((x * x).sum(-1, keepdims=True))
    y = x / np.maximum(n, 1e-12) * np.sqrt(x.shape[-1]) * g
    return y / (1.0 + np.exp(-y)) if silu else y


class VAEOracle:
    def __init__(self, P, z_dim, base_dim, dim_mult, num_res_blocks, temporal_upsample):
        self.P = P
        self.z_dim, self.dims = z_dim, dims_of(base_dim, dim_mult)
        self.n_up, self.nres, self.tup = len(dim_mult), num_res_blocks, temporal_upsample
        self.cache = {}

    def causal(self, name, x):
        w = self.P[name + ".w"]
        c = self.cache.get(name)
        if c is None:
            c = np.zeros((2,) + x.shape[1:])
        xin = np.concatenate([c, x], 0)
        self.cache[name] = xin[-2:].copy()
        kt = w.shape[2]
        return conv3d(xin[3 - kt:] if kt < 3 else xin, w, self.P[name + ".b"])

    def res(self, name, x):
        h = self.causal(name + ".conv1", rms(x, self.P[name + ".norm1.g"]))
        h = self.causal(name + ".conv2", rms(h, self.P[name + ".norm2.g"]))
        sc = x if (name + ".shortcut.w") not in self.P else conv3d(x, self.P[name + ".shortcut.w"],
                                                                   self.P[name + ".shortcut.b"])
        return h + sc

    def attn(self, name, x):
        """Mid-block attention, per frame: one head over the frame's h*w pixels,
        x + proj(softmax(q k^T / sqrt(C)) v) with q|k|v = rms(x) @ Wqkv^T + b (no SiLU)."""
        T, H, W, Cc = x.shape
        wq = self.P[name + ".qkv.w"][:, :, 0, 0, 0]
        wp = self.P[name + ".proj.w"][:, :, 0, 0, 0]
        out = x.copy()
        for t in range(T):
            u = rms(x[t], self.P[name + ".norm.g"], silu=False).reshape(-1, Cc)
            qkv = u @ wq.T + self.P[name + ".qkv.b"]
            q, k, v = qkv[:, :Cc], qkv[:, Cc:2 * Cc], qkv[:, 2 * Cc:]
            s = q @ k.T / np.sqrt(Cc)
            p = np.exp(s - s.max(1, keepdims=True))
            p /= p.sum(1, keepdims=True)
            out[t] += ((p @ v) @ wp.T + self.P[name + ".proj.b"]).reshape(H, W, Cc)
        return out

    def decode(self, z):
        """z [T, z_dim, h, w] -> frames [T*tf, 8h, 8w, 3] (float, pre-quantisation)."""
        x = np.transpose(np.asarray(z, dtype=np.float64), (0, 2, 3, 1))
        x = self.causal("conv_in", x)
        for j in range(2):
            x = self.res("mid.%d" % j, x)
            if j == 0 and "mid.attn.qkv.w" in self.P:
                x = self.attn("mid.attn", x)
        for i in range(self.n_up):
            for j in range(self.nres + 1):
                x = self.res("up.%d.res.%d" % (i, j), x)
            if i != self.n_up - 1:
                if self.tup[i]:
                    y = self.causal("up.%d.time" % i, x)          # [T, H, W, 2C]
                    C = y.shape[-1] // 2
                    x = np.stack([y[..., :C], y[..., C:]], 1).reshape(-1, *y.shape[1:3], C)
                x = x.repeat(2, axis=1).repeat(2, axis=2)
                x = conv3d(x, self.P["up.%d.resample.w" % i], self.P["up.%d.resample.b" % i])
        return self.causal("head.conv", rms(x, self.P["head.norm.g"]))


def to_rgb8(frames):
    return np.clip(np.rint((frames + 1.0) * 127.5), 0, 255).astype(np.uint8)
