"""CPU oracle (TEST INFRASTRUCTURE ONLY) for the "wan-shape" extension:
float64 NumPy restatement of the spatial-token DiT step with 3D RoPE and
AdaLN modulation/gating, plus the 2x2 patchify of the Eq.1 composite.

Parity status: PARTIALLY PINNED. The reference (`/root/reference/pkg`) has no
wan mode, so this file cannot be pinned to reference outputs as a whole.
What is pinned: every primitive it composes — sinusoid (net.py:200-206),
dense / layernorm / gelu / attention core (backends/reference.py:17-92),
composite layout (diffusion.py:150-179), sampler (diffusion.py:202-237) and
chunk geometry — is the same function `ftlk_oracle` restates and
`tests/test_oracle.py` pins to the reference's golden vectors at 1e-12. The
wan-specific composition (layer order with AdaLN: Wan-2.1 block structure;
RoPE split hd-4(hd//6) | 2(hd//6) | 2(hd//6); patch feature order
(c, py, px)) is builder-defined and documented in DESIGN.md.

Parameter layout: `paper_2512_23379_b200.config.param_shapes(mode="wan")`,
restated here by name only (weights are (in, out), applied x @ W + b).
"""

import numpy as np

from .ftlk_oracle import TIME_SCALE, dense, gelu, layernorm, sinusoid


def rope_split(hd):
    return (hd - 4 * (hd // 6)) // 2, (hd // 6), (hd // 6)


def rope_tables(frames, gh, gw, hd, theta=10000.0):
    pt, ph, pw = rope_split(hd)
    out = {}
    for ax, n, pairs in (("t", frames, pt), ("h", gh, ph), ("w", gw, pw)):
        inv = 1.0 / theta ** (np.arange(0, 2 * pairs, 2, dtype=np.float64) / (2 * pairs))
        ang = np.arange(n, dtype=np.float64)[:, None] * inv[None, :]
        out["cos_" + ax] = np.cos(ang).astype(np.float32)
        out["sin_" + ax] = np.sin(ang).astype(np.float32)
    return out


def apply_rope(x, tabs, gh, gw):
    """x: (L, H, hd) tokens frame-major then row then column."""
    L, H, hd = x.shape
    tok = np.arange(L)
    f, rem = tok // (gh * gw), tok % (gh * gw)
    yy, xx = rem // gw, rem % gw
    cos = np.concatenate([tabs["cos_t"][f], tabs["cos_h"][yy], tabs["cos_w"][xx]], axis=1).astype(np.float64)
    sin = np.concatenate([tabs["sin_t"][f], tabs["sin_h"][yy], tabs["sin_w"][xx]], axis=1).astype(np.float64)
    a, b = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = a * cos[:, None, :] - b * sin[:, None, :]
    out[..., 1::2] = a * sin[:, None, :] + b * cos[:, None, :]
    return out


def patchify(stacked, ph, pw):
    """(L_c, C, H, W) -> (L_c*(H/ph)*(W/pw), C*ph*pw), feature (c, py, px)."""
    lc, c, h, w = stacked.shape
    x = stacked.reshape(lc, c, h // ph, ph, w // pw, pw).transpose(0, 2, 4, 1, 3, 5)
    return x.reshape(lc * (h // ph) * (w // pw), c * ph * pw)


def unpatchify(tok, lc, d, h, w, ph, pw):
    x = tok.reshape(lc, h // ph, w // pw, d, ph, pw).transpose(0, 3, 1, 4, 2, 5)
    return x.reshape(lc, d, h, w)


def _head_attention(q, k, v, scale):
    s = (q @ k.T) * scale
    s -= s.max(axis=-1, keepdims=True)
    np.exp(s, out=s)
    s /= s.sum(axis=-1, keepdims=True)
    return s @ v


def attention(q, k, v, scale):
    """q (Lq, H, hd), k/v (Lk, H, hd) -> (Lq, H*hd). Softmax with max subtraction per head
    (backends/reference.py:84-89). One head at a time (an [H, Lq, Lk] score tensor is 35 GB at
    the 14B streaming shape); long sequences run the heads on a thread pool with single-threaded
    BLAS in each worker (NumPy's elementwise softmax is single-threaded, so this is ~8x faster
    than multithreaded BLAS one head after another; the arithmetic per head is unchanged)."""
    H = q.shape[1]
    o = np.empty((q.shape[0], H, v.shape[2]))
    if q.shape[0] * k.shape[0] < (1 << 22) or H == 1:
        for h in range(H):
            o[:, h] = _head_attention(q[:, h], k[:, h], v[:, h], scale)
        return o.reshape(q.shape[0], -1)
    import concurrent.futures as cf
    import os

    from threadpoolctl import threadpool_limits
    workers = max(1, min(H, os.cpu_count() or 1, 16))

    def one(h):
        o[:, h] = _head_attention(np.ascontiguousarray(q[:, h]), np.ascontiguousarray(k[:, h]),
                                  np.ascontiguousarray(v[:, h]), scale)
    with threadpool_limits(limits=1, user_api="blas"), cf.ThreadPoolExecutor(workers) as ex:
        list(ex.map(one, range(H)))
    return o.reshape(q.shape[0], -1)


def _rows_parallel(fn, x):
    """fn applied to row blocks of x on a thread pool (NumPy ufuncs release the GIL; the
    arithmetic per element is fn's). Used for the elementwise GELU over (L, ff) at 14B width."""
    import concurrent.futures as cf
    import os
    n = max(1, min(16, os.cpu_count() or 1))
    if x.shape[0] < 4096 or n == 1:
        return fn(x)
    out = np.empty_like(x)
    edges = np.linspace(0, x.shape[0], n + 1).astype(int)

    def one(i):
        out[edges[i]:edges[i + 1]] = fn(x[edges[i]:edges[i + 1]])
    with cf.ThreadPoolExecutor(n) as ex:
        list(ex.map(one, range(n)))
    return out


def silu(x):
    return x / (1.0 + np.exp(-x))


def composite_stacked(motion, z, reference):
    """Eq.1 stack (L_c, 2D+1, H, W): z_noise | z_mask | z_cond (diffusion.py:150-179)."""
    zn = np.concatenate([motion, z], axis=0)
    lc, d, h, w = zn.shape
    mask = np.zeros((lc, 1, h, w))
    mask[0] = 1.0
    cond = np.zeros_like(zn)
    cond[0] = reference
    return np.concatenate([zn, mask, cond], axis=1)


def denoise(P, cfg, motion, z, reference, audio, frame_t):
    """One wan-mode forward: x0 prediction (L_c, D, H, W).
    cfg: dict(model_dim, layers, heads, latent_dim, patch=(1,ph,pw), audio_tokens, audio_dim, rope_theta)."""
    m, heads, d = cfg["model_dim"], cfg["heads"], cfg["latent_dim"]
    hd = m // heads
    _, ph, pw = cfg["patch"]
    st = composite_stacked(motion, z, reference)
    lc, _, H, W = st.shape
    gh, gw = H // ph, W // pw
    T = gh * gw
    tok = patchify(st, ph, pw)
    L = tok.shape[0]
    frame_of = np.arange(L) // T
    h = dense(tok, P["in.w"], P["in.b"])
    temb = dense(sinusoid(np.asarray(frame_t) * TIME_SCALE, m), P["time.w"], P["time.b"])  # (L_c, m)
    e0 = dense(silu(temb), P["tproj.w"], P["tproj.b"]).reshape(lc, 6, m)
    pos = sinusoid(np.arange(lc), m)
    A = cfg["audio_tokens"]
    sig = dense(np.asarray(audio).reshape(lc * A, cfg["audio_dim"]), P["sig.w"], P["sig.b"]) + \
        np.repeat(pos, A, axis=0)
    ref = dense(np.asarray(reference).reshape(d, -1).mean(axis=1)[None], P["ref.w"], P["ref.b"])
    cond = np.vstack([sig, ref])
    tabs = rope_tables(lc, gh, gw, hd, cfg.get("rope_theta", 10000.0))
    scale = 1.0 / np.sqrt(hd)
    for i in range(cfg["layers"]):
        p = "layers.%d." % i
        mod = e0 + P[p + "mod"][None]            # (L_c, 6, m)
        mt = mod[frame_of]                       # (L, 6, m)
        xn, _, _ = layernorm(h, np.ones(m), np.zeros(m))
        u = xn * (1.0 + mt[:, 1]) + mt[:, 0]
        q = apply_rope((u @ P[p + "self.wq"]).reshape(L, heads, hd), tabs, gh, gw)
        k = apply_rope((u @ P[p + "self.wk"]).reshape(L, heads, hd), tabs, gh, gw)
        v = (u @ P[p + "self.wv"]).reshape(L, heads, hd)
        h = h + mt[:, 2] * (attention(q, k, v, scale) @ P[p + "self.wo"])
        u, _, _ = layernorm(h, P[p + "ln2.g"], P[p + "ln2.b"])
        cq = (u @ P[p + "cross.wq"]).reshape(L, heads, hd)
        ck = (cond @ P[p + "cross.wk"]).reshape(-1, heads, hd)
        cv = (cond @ P[p + "cross.wv"]).reshape(-1, heads, hd)
        h = h + attention(cq, ck, cv, scale) @ P[p + "cross.wo"]
        xn, _, _ = layernorm(h, np.ones(m), np.zeros(m))
        u = xn * (1.0 + mt[:, 4]) + mt[:, 3]
        f = dense(_rows_parallel(gelu, dense(u, P[p + "ffn.w1"], P[p + "ffn.b1"])), P[p + "ffn.w2"], P[p + "ffn.b2"])
        h = h + mt[:, 5] * f
    fm = P["final.mod"][None] + temb[:, None, :]  # (L_c, 2, m)
    ft = fm[frame_of]
    xn, _, _ = layernorm(h, np.ones(m), np.zeros(m))
    u = xn * (1.0 + ft[:, 1]) + ft[:, 0]
    out = dense(u, P["out.w"], P["out.b"])
    return unpatchify(out, lc, d, H, W, ph, pw)


def sample_chunk(P, cfg, timesteps, motion, reference, audio, z0, trace=None):
    """DDIM ladder (diffusion.py:202-237) around the wan-mode forward."""
    lm = motion.shape[0]
    z = np.array(z0, dtype=np.float64)
    lc = lm + z.shape[0]
    x0 = None
    ts = list(timesteps)
    for i, t in enumerate(ts):
        frame_t = np.where(np.arange(lc) < lm, 0.0, float(t))
        x0 = denoise(P, cfg, motion, z, reference, audio, frame_t)[lm:]
        if trace is not None:
            trace.append((t, z.copy(), x0.copy()))
        if i + 1 < len(ts):
            eps = (z - (1.0 - t) * x0) / t
            tn = ts[i + 1]
            z = (1.0 - tn) * x0 + tn * eps
    return np.concatenate([motion, x0], axis=0)
