"""3D rotary position tables (wan mode), computed on the host in float64.

Head dim hd is split Wan-style into a frame axis of hd - 4*(hd//6) dims and
row / column axes of 2*(hd//6) dims each; each axis a of width d_a uses
frequencies theta^(-2i/d_a), i < d_a/2, and rotates consecutive pairs
(x[2p], x[2p+1]) by pos * freq. Positions are chunk-relative latent frame
index (as the reference's chunk-relative sinusoid positions, net.py:228) and
the token's row / column in the patch grid.

The tables are the bit-exact contract of the north star: they are computed
once here in float64 and rounded to float32 for upload; the device never
recomputes them (tests compare the uploaded bytes to the oracle's tables).
"""

import numpy as np


def rope_split(hd: int):
    hd_t = hd - 4 * (hd // 6)
    hd_s = 2 * (hd // 6)
    return hd_t // 2, hd_s // 2, hd_s // 2


def axis_angles(n_pos: int, dim: int, theta: float) -> np.ndarray:
    inv = 1.0 / (theta ** (np.arange(0, dim, 2, dtype=np.float64) / dim))
    return np.arange(n_pos, dtype=np.float64)[:, None] * inv[None, :]


def rope3d_tables(frames: int, grid_h: int, grid_w: int, hd: int, theta: float = 10000.0) -> dict:
    pt, ph, pw = rope_split(hd)
    out = {}
    for ax, n, pairs in (("t", frames, pt), ("h", grid_h, ph), ("w", grid_w, pw)):
        ang = axis_angles(n, 2 * pairs, theta)
        out["cos_" + ax] = np.cos(ang).astype(np.float32)
        out["sin_" + ax] = np.sin(ang).astype(np.float32)
    return out


def per_token_tables(tables: dict, grid_h: int, grid_w: int):
    """Per-axis tables -> per-token float32 [frames*grid_h*grid_w][hd/2] cos and sin
    (token order frame-major, then row, then column); a pure gather of the
    float32-rounded per-axis values, so it stays bit-identical to them."""
    frames = tables["cos_t"].shape[0]
    f = np.repeat(np.arange(frames), grid_h * grid_w)
    y = np.tile(np.repeat(np.arange(grid_h), grid_w), frames)
    x = np.tile(np.arange(grid_w), frames * grid_h)
    cos = np.concatenate([tables["cos_t"][f], tables["cos_h"][y], tables["cos_w"][x]], axis=1)
    sin = np.concatenate([tables["sin_t"][f], tables["sin_h"][y], tables["sin_w"][x]], axis=1)
    return np.ascontiguousarray(cos, dtype=np.float32), np.ascontiguousarray(sin, dtype=np.float32)
