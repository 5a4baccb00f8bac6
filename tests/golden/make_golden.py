"""Freeze golden vectors by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference package `ftlk` in place from /root/reference (read-only)
and writes `tests/golden/ftlk_golden.npz`. Nothing else reads /root/reference:
the GPU box never has it, so the frozen arrays are what tests compare to.

What is frozen (reference call sites in parentheses):
  k_*     operator table I/O, NumPy backend (backends/reference.py:17-92)
  p_*     ParamStore.init checksums (net.py:99-112, :132-137)
  f_*     Denoiser.forward on seeded composites (net.py:240-276)
  s_*     few_step_sample with trace, 4/2/1-step ladders (diffusion.py:202-237)
  r_*     rollout_stream over 5 chunks + Codec.decode (metrics.py:128-149, world.py:206-210)
  e_*     threaded StreamSession (streaming.py:123-356): emitted indices/states
  w_*     chunk windows incl. pre-roll and motion_len=0 geometry (streaming.py:259-270)
  r_P/r_w world identity injection and mouth readout (world.py:76-120) for the server tests
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("FTLK_BACKEND", "python")

from ftlk import backends as B  # noqa: E402
from ftlk.diffusion import SamplerPlan, composite_from_state, few_step_sample  # noqa: E402
from ftlk.metrics import NetGenerator, make_stream_context, rollout_stream  # noqa: E402
from ftlk.net import Denoiser, NetConfig, ParamStore  # noqa: E402
from ftlk.streaming import StreamConfig, start_stream  # noqa: E402
from ftlk.world import Codec, World, WorldSpec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ftlk_golden.npz")


def main():
    g = {"numpy_version": np.array(np.__version__), "backend": np.array(B.active_backend())}
    ref = B.get_backend("python")
    rng = np.random.default_rng(0)

    # ---- operator table
    x, w, b = rng.standard_normal((7, 5)), rng.standard_normal((5, 3)), rng.standard_normal(3)
    g.update(k_dense_x=x, k_dense_w=w, k_dense_b=b, k_dense_y=ref.dense_forward(x, w, b))
    x = rng.standard_normal((6, 8)) * 3.0
    g.update(k_gelu_x=x, k_gelu_y=ref.gelu_forward(x))
    x, ga, be = rng.standard_normal((6, 8)) + 2.0, rng.standard_normal(8), rng.standard_normal(8)
    y, mu, rs = ref.layernorm_forward(x, ga, be)
    g.update(k_ln_x=x, k_ln_g=ga, k_ln_b=be, k_ln_y=y, k_ln_mean=mu, k_ln_rstd=rs)
    for heads in (1, 2, 4):
        for cross in (0, 1):
            m = 8
            xq = rng.standard_normal((5, m))
            xkv = rng.standard_normal((3, m)) if cross else xq
            ws = [rng.standard_normal((m, m)) for _ in range(4)]
            yy, cache = ref.mha_forward(xq, xkv, *ws, heads)
            key = "k_mha_h%d_c%d_" % (heads, cross)
            g[key + "xq"], g[key + "xkv"] = xq, xkv
            for nm, arr in zip(("wq", "wk", "wv", "wo"), ws):
                g[key + nm] = arr
            g[key + "y"], g[key + "p"] = yy, cache[3]

    # ---- params
    cfgs = {"default": (NetConfig(), 200), "tiny": (NetConfig(8, 1, 2, 16, 4), 0),
            "h4": (NetConfig(32, 2, 4, 48, 8), 7)}
    stores = {}
    for name, (cfg, seed) in cfgs.items():
        st = ParamStore.init(cfg, seed)
        stores[name] = st
        g["p_%s_checksum" % name] = np.array(st.checksum())
        g["p_%s_n" % name] = np.array(st.n_params)

    # ---- denoiser forward
    for name, (cfg, _) in cfgs.items():
        net = Denoiser(cfg)
        r = np.random.default_rng(11)
        d = cfg.latent_dim
        for lm, t in ((2, 0.75), (0, 1.0), (3, 0.25)):
            lc = 9 if lm != 3 else 7
            motion = r.standard_normal((lm, d))
            z = r.standard_normal((lc - lm, d))
            refl = r.standard_normal(d)
            sig = r.uniform(-1, 1, lc)
            comp = composite_from_state(motion, z, refl, sig, t)
            key = "f_%s_lm%d_" % (name, lm)
            g[key + "motion"], g[key + "z"], g[key + "ref"], g[key + "sig"] = motion, z, refl, sig
            g[key + "t"] = np.array(t)
            g[key + "stacked"] = comp.stacked()
            g[key + "frame_t"] = comp.frame_t
            g[key + "out"] = net.forward(stores[name], comp)

    # ---- sampler with trace
    cfg = cfgs["default"][0]
    fn = Denoiser(cfg).as_denoise_fn(stores["default"])
    r = np.random.default_rng(12)
    motion, refl, sig = r.standard_normal((2, 8)), r.standard_normal(8), r.uniform(-1, 1, 9)
    g.update(s_motion=motion, s_ref=refl, s_sig=sig)
    for plan in (SamplerPlan(), SamplerPlan(2, (1.0, 0.5)), SamplerPlan(1, (1.0,))):
        tr = []
        from ftlk.seeding import STREAM_NOISE, rng_for
        chunk = few_step_sample(fn, plan, motion, refl, sig, rng_for(5, STREAM_NOISE, 3), trace=tr)
        key = "s_steps%d_" % plan.steps
        g[key + "timesteps"] = np.array(plan.timesteps)
        g[key + "latents"] = chunk.latents
        g[key + "z"] = np.stack([t[1] for t in tr])
        g[key + "x0"] = np.stack([t[2] for t in tr])

    # ---- rollout + decode
    world = World(WorldSpec())
    codec = Codec.for_world(world)
    ctx = make_stream_context(world, codec, 3, 0, 35)
    gen = NetGenerator(stores["default"], cfg, SamplerPlan())
    targets, motions = rollout_stream(gen, ctx, 35)
    # world readouts for the WebSocket front door (world.py:76-120): identity injection P, mouth w
    from ftlk.world import sample_identity
    g.update(r_P=world.P, r_w=world.w, r_identity=sample_identity(1, world.spec.identity_dim))
    g.update(r_Q=world.Q, r_seed=np.array(ctx.seed, dtype=np.uint64), r_signal=ctx.signal,
             r_reference_latent=ctx.reference_latent, r_reference_frame=ctx.reference_frame,
             r_targets=targets, r_motions=np.stack(motions), r_frames=codec.decode(targets))

    # ---- threaded engine (same geometry as rollout)
    scfg = StreamConfig(seed=int(ctx.seed))
    sess = start_stream(stores["default"], cfg, codec, ctx.reference_frame, scfg)
    sess.push_signal((i, ctx.signal[i]) for i in range(35))
    got = []
    import time
    deadline = time.time() + 60
    while len(got) < 35 and time.time() < deadline:
        fr, _ = sess.next_frames(wait=True, timeout=0.2)
        got.extend(fr)
    sess.close()
    g["e_index"] = np.array([f.index for f in got])
    g["e_chunk"] = np.array([f.chunk for f in got])
    g["e_state"] = np.stack([f.state for f in got])

    # ---- window geometry incl. pre-roll, motion_len = 0, long chunks
    sig = np.arange(1, 41, dtype=np.float64) / 50.0
    for lc, lm in ((9, 2), (5, 0), (6, 5)):
        wins = []
        for c in range(4):
            lo = c * (lc - lm) - lm
            wins.append([sig[j] if 0 <= j < len(sig) else 0.0 for j in range(lo, lo + lc)])
        g["w_%d_%d" % (lc, lm)] = np.array(wins)
    g["w_signal"] = sig

    # ---- FTLK checkpoint written by the reference writer (checkpoint.py:31-53)
    from ftlk.checkpoint import save as ref_save
    ref_save(os.path.join(os.path.dirname(OUT), "tiny.ftlk"), stores["tiny"], "generator_student",
             cfgs["tiny"][0])
    g["c_tiny_checksum"] = np.array(stores["tiny"].checksum())

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, len(g), "arrays")


if __name__ == "__main__":
    main()
