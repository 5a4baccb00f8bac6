"""CPU oracle (TEST INFRASTRUCTURE ONLY) — float64 NumPy restatement of the
reference streaming hot path in "ftlk" mode.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module, and only as the checker or
the timed CPU baseline. The product package never imports it.

Parity pin: every function here is checked against golden vectors produced by
running the reference itself (`tests/golden/make_golden.py` imports
`/root/reference/pkg/src/ftlk` in the build container and freezes
`tests/golden/ftlk_golden.npz`); `tests/test_oracle.py` holds the pins at
rtol=atol=1e-12 (the reference's own backend tolerance,
`pkg/tests/test_backends.py:17`).

Restated reference functions (file:line under /root/reference/pkg/src/ftlk):
  rng_for ............... seeding.py:26-36
  sinusoid .............. net.py:200-206
  init_params ........... net.py:56-85 (shapes), net.py:99-112 (init)
  dense/gelu/layernorm .. backends/reference.py:17-18, :28-31, :41-46
  mha ................... backends/reference.py:62-92
  embed ................. net.py:223-238
  denoise ............... net.py:244-276
  composite ............. diffusion.py:150-179 (+ stacked, :133-135)
  sample_chunk .......... diffusion.py:202-237
  stream windows ........ streaming.py:259-270, metrics.py:140-143
  rollout ............... metrics.py:128-149 (engine twin, streaming.py:283-306)
  codec decode/encode ... world.py:200-210
"""

import numpy as np

TIME_SCALE = 1000.0
LN_EPS = 1e-6
GELU_C = np.sqrt(2.0 / np.pi)
GELU_A = 0.044715
STREAM_NOISE = 9
INIT = 4


# ---------------------------------------------------------------- RNG
def rng_for(seed, *tags):
    path = []

    def walk(x):
        if isinstance(x, (list, tuple)):
            for y in x:
                walk(y)
        else:
            path.append(int(x) & 0xFFFFFFFFFFFFFFFF)

    walk((seed,) + tags)
    return np.random.default_rng(np.random.SeedSequence(path))


# ---------------------------------------------------------------- tables
def sinusoid(positions, dim):
    """[sin | cos] features, frequency denominator max(half-1, 1)."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1)
    half = dim // 2
    k = np.arange(half, dtype=np.float64)
    freq = np.exp(-np.log(10000.0) * k / max(half - 1, 1))
    arg = np.outer(pos, freq)
    out = np.empty((pos.shape[0], 2 * half))
    out[:, :half] = np.sin(arg)
    out[:, half:] = np.cos(arg)
    return out


# ---------------------------------------------------------------- params
def ftlk_shapes(m, layers, ff, d):
    s = [("in.w", (2 * d + 1, m)), ("in.b", (m,)), ("time.w", (m, m)), ("time.b", (m,)),
         ("sig.w", (1, m)), ("sig.b", (m,)), ("ref.w", (d, m)), ("ref.b", (m,))]
    for i in range(layers):
        p = "layers.%d." % i
        for nm, sh in (("ln1.g", (m,)), ("ln1.b", (m,)),
                       ("self.wq", (m, m)), ("self.wk", (m, m)), ("self.wv", (m, m)), ("self.wo", (m, m)),
                       ("ln2.g", (m,)), ("ln2.b", (m,)),
                       ("cross.wq", (m, m)), ("cross.wk", (m, m)), ("cross.wv", (m, m)), ("cross.wo", (m, m)),
                       ("ln3.g", (m,)), ("ln3.b", (m,)),
                       ("ffn.w1", (m, ff)), ("ffn.b1", (ff,)), ("ffn.w2", (ff, m)), ("ffn.b2", (m,))):
            s.append((p + nm, sh))
    s += [("final.g", (m,)), ("final.b", (m,)), ("out.w", (m, d)), ("out.b", (d,))]
    return s


def init_params(shapes, seed):
    """Gains 1, biases / 1-d tensors 0, matrices N(0,1)/sqrt(fan_in) drawn in
    order from one (seed, INIT) stream."""
    g = rng_for(seed, INIT)
    out = {}
    for name, shape in shapes:
        if name.endswith(".g"):
            out[name] = np.ones(shape)
        elif name.endswith(".b") or len(shape) == 1:
            out[name] = np.zeros(shape)
        else:
            out[name] = g.standard_normal(shape) / np.sqrt(shape[0])
    return out


# ---------------------------------------------------------------- kernels
def dense(x, w, b):
    return np.asarray(x) @ np.asarray(w) + np.asarray(b)


def gelu(x):
    x = np.asarray(x)
    return 0.5 * x * (1.0 + np.tanh(GELU_C * (x + GELU_A * x ** 3)))


def layernorm(x, g, b):
    x = np.asarray(x)
    mu = x.mean(axis=1)
    var = ((x - mu[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    return ((x - mu[:, None]) * rstd[:, None]) * g + b, mu, rstd


def softmax_rows(s):
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def mha(xq, xkv, wq, wk, wv, wo, heads):
    """Returns (y, (q, k, v, p, ctx)) with q/k/v as (H, n, hd)."""
    n, m = xq.shape
    hd = m // heads

    def split(t):
        return t.reshape(t.shape[0], heads, hd).transpose(1, 0, 2)

    q, k, v = split(xq @ wq), split(xkv @ wk), split(xkv @ wv)
    p = softmax_rows(np.einsum("hid,hjd->hij", q, k) / np.sqrt(hd))
    ctx = np.einsum("hij,hjd->hid", p, v).transpose(1, 0, 2).reshape(n, m)
    return ctx @ wo, (q, k, v, p, ctx)


# ---------------------------------------------------------------- model
def composite(motion, z, reference, signal, t):
    """Eq.1 assembly: returns dict with stacked (L_c, 2D+1) and frame_t."""
    motion = np.atleast_2d(np.asarray(motion, dtype=np.float64))
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    d = z.shape[1]
    if motion.size == 0:
        motion = motion.reshape(0, d)
    lm = motion.shape[0]
    lc = lm + z.shape[0]
    z_noise = np.vstack([motion, z])
    mask = np.zeros((lc, 1))
    mask[0, 0] = 1.0
    cond = np.zeros((lc, d))
    cond[0] = reference
    frame_t = np.where(np.arange(lc) < lm, 0.0, float(t))
    return {"stacked": np.hstack([z_noise, mask, cond]), "frame_t": frame_t,
            "signal": np.asarray(signal, dtype=np.float64),
            "reference": np.asarray(reference, dtype=np.float64), "motion_len": lm}


def embed(P, m, comp):
    lc = comp["stacked"].shape[0]
    pos = sinusoid(np.arange(lc), m)
    tfeat = sinusoid(comp["frame_t"] * TIME_SCALE, m)
    h = dense(comp["stacked"], P["in.w"], P["in.b"]) + dense(tfeat, P["time.w"], P["time.b"]) + pos
    sig = dense(comp["signal"][:, None], P["sig.w"], P["sig.b"]) + pos
    ref = dense(comp["reference"][None, :], P["ref.w"], P["ref.b"])
    return h, np.vstack([sig, ref])


def denoise(P, cfg, comp):
    """Full-chunk x0 prediction (L_c, D). cfg: dict(model_dim, layers, heads)."""
    m, heads = cfg["model_dim"], cfg["heads"]
    h, cond = embed(P, m, comp)
    for i in range(cfg["layers"]):
        p = "layers.%d." % i
        u, _, _ = layernorm(h, P[p + "ln1.g"], P[p + "ln1.b"])
        h = h + mha(u, u, P[p + "self.wq"], P[p + "self.wk"], P[p + "self.wv"], P[p + "self.wo"], heads)[0]
        u, _, _ = layernorm(h, P[p + "ln2.g"], P[p + "ln2.b"])
        h = h + mha(u, cond, P[p + "cross.wq"], P[p + "cross.wk"], P[p + "cross.wv"], P[p + "cross.wo"], heads)[0]
        u, _, _ = layernorm(h, P[p + "ln3.g"], P[p + "ln3.b"])
        h = h + dense(gelu(dense(u, P[p + "ffn.w1"], P[p + "ffn.b1"])), P[p + "ffn.w2"], P[p + "ffn.b2"])
    u, _, _ = layernorm(h, P["final.g"], P["final.b"])
    return dense(u, P["out.w"], P["out.b"])


def sample_chunk(denoise_fn, timesteps, motion, reference, signal, rng=None, z0=None, trace=None):
    """DDIM recursion over the ladder; alpha = 1 - t, sigma = t.
    Returns the chunk latents [motion; x0_last] (L_c, D)."""
    reference = np.asarray(reference, dtype=np.float64)
    signal = np.asarray(signal, dtype=np.float64)
    d = reference.shape[0]
    motion = np.atleast_2d(np.asarray(motion, dtype=np.float64))
    if motion.size == 0:
        motion = motion.reshape(0, d)
    n_t = signal.shape[0] - motion.shape[0]
    z = rng.standard_normal((n_t, d)) if z0 is None else np.array(z0, dtype=np.float64)
    x0 = None
    ts = list(timesteps)
    for i, t in enumerate(ts):
        x0 = denoise_fn(composite(motion, z, reference, signal, t))[motion.shape[0]:]
        if trace is not None:
            trace.append((t, z.copy(), x0.copy()))
        if i + 1 < len(ts):
            eps = (z - (1.0 - t) * x0) / t
            tn = ts[i + 1]
            z = (1.0 - tn) * x0 + tn * eps
    return np.vstack([motion, x0])


def window_indices(c, chunk_len, motion_len):
    lo = c * (chunk_len - motion_len) - motion_len
    return np.arange(lo, lo + chunk_len)


def window(signal, c, chunk_len, motion_len):
    """Driving window of chunk c; indices outside [0, len) read 0.0."""
    idx = window_indices(c, chunk_len, motion_len)
    sig = np.asarray(signal, dtype=np.float64)
    ok = (idx >= 0) & (idx < sig.shape[0])
    out = np.zeros(idx.shape[0])
    out[ok] = sig[idx[ok]]
    return out


def rollout(denoise_fn, timesteps, reference_latent, signal, n_frames, seed,
            chunk_len=9, motion_len=2, motion_override=None):
    """Synchronous generate: returns (targets (n_frames, D), motions per chunk,
    emitted frame indices). `motion_override[c]`, if given, teacher-forces
    the motion rows of chunk c."""
    stride = chunk_len - motion_len
    n_chunks = int(np.ceil(n_frames / stride))
    motion = np.repeat(np.asarray(reference_latent, dtype=np.float64)[None, :], motion_len, axis=0)
    outs, motions, idx = [], [], []
    for c in range(n_chunks):
        if motion_override is not None:
            motion = motion_override[c]
        lat = sample_chunk(denoise_fn, timesteps, motion, reference_latent,
                           window(signal, c, chunk_len, motion_len),
                           rng_for(seed, STREAM_NOISE, c))
        motions.append(motion)
        outs.append(lat[motion_len:])
        idx.extend(c * stride + j for j in range(stride))
        if motion_len:
            motion = lat[-motion_len:]
    return np.vstack(outs)[:n_frames], motions, np.asarray(idx[:n_frames])


def codec_decode(latents, Q):
    return np.asarray(latents) @ Q


def codec_encode(frames, Q):
    return np.asarray(frames) @ Q.T
