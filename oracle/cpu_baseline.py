"""CPU baseline (TEST/BENCH INFRASTRUCTURE ONLY): times the float64 NumPy
oracle of the hot path on the host cores, for bench.py's `cpu_baseline` leg
and its `--impl reference` arm.

The reference's own path is NumPy float64 on CPU (`pkg/src/ftlk/net.py` +
`backends/reference.py`); at the 14B shape (m=5120, 40 heads, 40 layers,
L=10530 tokens) one chunk is infeasible on a host (fp64 weights 105 GiB, one
attention-probability tensor 35.5 GB). The bounded sample is one
wan-shaped layer forward (AdaLN + self-attention + cross-attention + FFN, the
same ops as `wan_oracle.denoise`) at the full model width on `L_s` tokens
(default one latent frame, 1 170 tokens at 416x720), timed split into its
token-linear part and its attention part. The self-attention core (the
reference's einsum form, backends/reference.py:84-89, single-threaded NumPy)
is timed on `attn_heads` of the heads (every head costs the same) and scaled
by heads / attn_heads; the chunk time is extrapolated as
    layers * steps * (t_lin * L/L_s + t_attn * (L/L_s)^2)
and reported as an EXTRAPOLATED baseline with the method stated.
"""

import os
import time

import numpy as np

from .ftlk_oracle import gelu, layernorm


def _rand(rng, shape, fan_in):
    return rng.standard_normal(shape) / np.sqrt(fan_in)


def make_layer(m, ff, seed=0):
    r = np.random.default_rng(seed)
    P = {k: _rand(r, (m, m), m) for k in ("wq", "wk", "wv", "wo", "cq", "ck", "cv", "co")}
    P["w1"], P["b1"] = _rand(r, (m, ff), m), np.zeros(ff)
    P["w2"], P["b2"] = _rand(r, (ff, m), ff), np.zeros(m)
    P["mod"] = _rand(r, (6, m), m)
    P["ln2g"], P["ln2b"] = np.ones(m), np.zeros(m)
    return P


def _attn(q, k, v, heads):
    L, m = q.shape
    hd = m // heads
    qh, kh, vh = (x.reshape(-1, heads, hd).transpose(1, 0, 2) for x in (q, k, v))
    s = np.einsum("hqd,hkd->hqk", qh, kh) / np.sqrt(hd)
    s -= s.max(-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(-1, keepdims=True)
    return np.einsum("hqk,hkd->hqd", p, vh).transpose(1, 0, 2).reshape(L, m)


def layer_timed(P, h, cond, heads, attn_heads=None):
    """One wan layer (wan_oracle.denoise inner block, without RoPE's table
    gather cost) -> (h_out, t_linear_s, t_attention_s). attn_heads: time the
    self-attention core on that many heads and scale to all (the others' output
    columns reuse the timed heads' values; cost per head is identical)."""
    m = h.shape[1]
    ones, zeros = np.ones(m), np.zeros(m)
    mod = P["mod"]
    t0 = time.perf_counter()
    u = layernorm(h, ones, zeros)[0] * (1 + mod[1]) + mod[0]
    q, k, v = u @ P["wq"], u @ P["wk"], u @ P["wv"]
    t1 = time.perf_counter()
    ah = heads if not attn_heads or attn_heads >= heads else int(attn_heads)
    hd = m // heads
    sub = _attn(q[:, :ah * hd], k[:, :ah * hd], v[:, :ah * hd], ah)
    a = np.tile(sub, (1, heads // ah + 1))[:, :m]
    t2 = time.perf_counter()
    t_att = (t2 - t1) * heads / ah
    h = h + mod[2] * (a @ P["wo"])
    u = layernorm(h, P["ln2g"], P["ln2b"])[0]
    h = h + _attn(u @ P["cq"], cond @ P["ck"], cond @ P["cv"], heads) @ P["co"]
    u = layernorm(h, ones, zeros)[0] * (1 + mod[4]) + mod[3]
    h = h + mod[5] * (gelu(u @ P["w1"] + P["b1"]) @ P["w2"] + P["b2"])
    t3 = time.perf_counter()
    return h, (t1 - t0) + (t3 - t2), t_att


def extrapolated_chunk_seconds(m=5120, heads=40, ff=13824, layers=40, steps=4, L=10530, L_s=1170, n_cond=37,
                               reps=1, seed=0, P=None, attn_heads=4):
    """Returns (chunk_seconds, detail dict)."""
    P = P if P is not None else make_layer(m, ff, seed)
    r = np.random.default_rng(seed + 1)
    h = r.standard_normal((L_s, m))
    cond = r.standard_normal((n_cond, m))
    tl, ta = [], []
    for _ in range(reps):
        _, a, b = layer_timed(P, h, cond, heads, attn_heads)
        tl.append(a)
        ta.append(b)
    t_lin, t_att = float(np.median(tl)), float(np.median(ta))
    f = L / L_s
    per_layer = t_lin * f + t_att * f * f
    chunk = per_layer * layers * steps
    return chunk, {"t_linear_s": t_lin, "t_attention_s": t_att, "L_sample": L_s, "L": L,
                   "per_layer_s": per_layer, "layers": layers, "steps": steps, "attn_heads_timed": attn_heads,
                   "heads": heads, "threads": os.cpu_count()}
