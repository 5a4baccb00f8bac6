"""Model-level parity on the B200: the device denoiser / sampler against the
reference's own outputs (ftlk mode, golden vectors) and against the float64
oracle (wan mode). Bar: relative L2 <= 1e-2 (north star bf16 budget)."""

import numpy as np
import pytest

from oracle import ftlk_oracle as FO
from oracle import wan_oracle as WO

pytestmark = pytest.mark.gpu
BUDGET = 1e-2


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


CFGS = {"default": ((32, 2, 2, 64, 8), 200), "tiny": ((8, 1, 2, 16, 4), 0), "h4": ((32, 2, 4, 48, 8), 7)}


def _store(name):
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    (m, layers, heads, ff, d), seed = CFGS[name]
    cfg = NetConfig(m, layers, heads, ff, d)
    return cfg, ParamStore.init(cfg, seed)


@pytest.mark.parametrize("name", list(CFGS))
@pytest.mark.parametrize("lm", [2, 0, 3])
def test_ftlk_forward_matches_reference(golden, cuda, name, lm):
    from paper_2512_23379_b200.diffusion import composite_from_state
    from paper_2512_23379_b200.net import Denoiser
    cfg, store = _store(name)
    k = "f_%s_lm%d_" % (name, lm)
    comp = composite_from_state(golden[k + "motion"], golden[k + "z"], golden[k + "ref"], golden[k + "sig"],
                                float(golden[k + "t"]))
    out = Denoiser(cfg).forward(store, comp)
    assert out.shape == golden[k + "out"].shape
    assert rel(out, golden[k + "out"]) < BUDGET
    # same bf16-rounded weights in the fp64 oracle: isolates kernel arithmetic error
    P = store.bf16_rounded().params
    ocfg = dict(model_dim=cfg.model_dim, layers=cfg.layers, heads=cfg.heads)
    ref = FO.denoise(P, ocfg, FO.composite(golden[k + "motion"], golden[k + "z"], golden[k + "ref"],
                                            golden[k + "sig"], float(golden[k + "t"])))
    assert rel(out, ref) < 5e-3


@pytest.mark.parametrize("steps", [4, 2, 1])
def test_ftlk_sampler_matches_reference(golden, cuda, steps):
    from paper_2512_23379_b200.config import SamplerPlan
    from paper_2512_23379_b200.diffusion import few_step_sample
    from paper_2512_23379_b200.net import Denoiser
    from paper_2512_23379_b200.seeding import STREAM_NOISE, rng_for
    cfg, store = _store("default")
    k = "s_steps%d_" % steps
    plan = SamplerPlan(steps, tuple(golden[k + "timesteps"]))
    tr = []
    chunk = few_step_sample(Denoiser(cfg).as_denoise_fn(store), plan, golden["s_motion"], golden["s_ref"],
                            golden["s_sig"], rng_for(5, STREAM_NOISE, 3), trace=tr)
    g = golden[k + "latents"]
    assert np.array_equal(chunk.latents[:2], g[:2])               # motion rows carried exactly
    assert rel(chunk.targets, g[2:]) < BUDGET
    assert rel(tr[0][1], golden[k + "z"][0]) < 1e-7               # host PCG64 draw, fp32 sampler state
    for i in range(steps):
        assert rel(tr[i][2], golden[k + "x0"][i]) < BUDGET


WAN_CASES = {
    # m, layers, heads, ff, D, A, adim, Lc, Lm, H, W
    "hd128": (256, 2, 2, 512, 16, 2, 32, 3, 1, 16, 24),
    "hd64": (256, 2, 4, 384, 16, 4, 16, 4, 2, 12, 20),
    "hd64_small": (128, 1, 2, 256, 4, 1, 8, 2, 1, 4, 6),
}


def _wan(case, seed=3):
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    m, layers, heads, ff, D, A, adim, Lc, Lm, H, W = WAN_CASES[case]
    cfg = NetConfig(m, layers, heads, ff, D, mode="wan", patch=(1, 2, 2), audio_dim=adim, audio_tokens=A)
    store = ParamStore.init(cfg, seed)
    r = np.random.default_rng(seed)
    inputs = dict(motion=r.standard_normal((Lm, D, H, W)), z=r.standard_normal((Lc - Lm, D, H, W)),
                  ref=r.standard_normal((D, H, W)), audio=r.standard_normal((Lc, A, adim)))
    ocfg = dict(model_dim=m, layers=layers, heads=heads, latent_dim=D, patch=(1, 2, 2), audio_tokens=A,
                audio_dim=adim)
    return cfg, store, inputs, ocfg


@pytest.mark.parametrize("case", list(WAN_CASES))
def test_wan_forward_matches_oracle(cuda, case):
    from paper_2512_23379_b200.diffusion import composite_from_state
    from paper_2512_23379_b200.net import Denoiser
    cfg, store, x, ocfg = _wan(case)
    comp = composite_from_state(x["motion"], x["z"], x["ref"], x["audio"], 0.75)
    out = Denoiser(cfg).forward(store, comp)
    P = store.bf16_rounded().params
    ref = WO.denoise(P, ocfg, x["motion"], x["z"], x["ref"], x["audio"], comp.frame_t)
    assert out.shape == ref.shape
    assert rel(out, ref) < BUDGET


def test_wan_sampler_matches_oracle(cuda):
    from paper_2512_23379_b200.config import SamplerPlan
    from paper_2512_23379_b200.diffusion import few_step_sample
    from paper_2512_23379_b200.net import Denoiser
    from paper_2512_23379_b200.seeding import STREAM_NOISE, rng_for
    cfg, store, x, ocfg = _wan("hd128")
    chunk = few_step_sample(Denoiser(cfg).as_denoise_fn(store), SamplerPlan(), x["motion"], x["ref"], x["audio"],
                            rng_for(11, STREAM_NOISE, 0))
    z0 = rng_for(11, STREAM_NOISE, 0).standard_normal(x["z"].shape)
    ref = WO.sample_chunk(store.bf16_rounded().params, ocfg, (1.0, 0.75, 0.5, 0.25), x["motion"], x["ref"],
                          x["audio"], z0)
    assert np.array_equal(chunk.latents[:1], x["motion"])
    assert rel(chunk.targets, ref[1:]) < BUDGET


def test_wan_folded_cross_attention_matches_projections(cuda):
    """Cross-attention folded through the chunk's fixed K/V (S = U.(s Wq K^T), out = P.(V Wo),
    the fold as two block-diagonal tensor-core GEMMs with the K-band skip) == the explicit
    Q projection -> attention -> O projection path; the folded operands At / Bt == their fp32
    definition from the device cond K/V."""
    import torch

    from paper_2512_23379_b200 import ops
    from paper_2512_23379_b200.model import DeviceDenoiser, DeviceWeights
    cfg, store, x, ocfg = _wan("hd128")
    Lc, Lm = x["audio"].shape[0], x["motion"].shape[0]
    H, W = x["ref"].shape[1:]
    w = DeviceWeights.from_host(cfg, store.params, cuda)
    outs = []
    for fold, band in ((True, True), (False, True), (True, False)):
        d = DeviceDenoiser(w, Lc, Lm, (H, W), fold_cross=fold, fold_band=band)
        assert d.fold == fold
        d.prepare_cond(x["audio"], x["ref"])
        fv = d.frame_vectors(np.where(np.arange(Lc) < Lm, 0.0, 0.75))
        args = [torch.as_tensor(x[k], dtype=torch.float32, device=cuda) for k in ("motion", "z", "ref")]
        outs.append(d.tokens_to_frames(d.step(*args, fv)).double().cpu().numpy())
        if fold and band:
            m, hd, J, nc = cfg.model_dim, cfg.head_dim, d.J, d.n_cond
            at = d.buf["xat"].float()[:, ops.tiled_seg_rows(cfg.heads, J).to(cuda)]   # [layers, H*J, m]
            bt = d.buf["xbt"].float()                                                   # [layers, m, H*J]
            for i in range(cfg.layers):
                kv = d.buf["ckv"][i].float()
                wq = w.cross_wq_io(i).float()                                  # (in, out)
                wo_t = w.mats["layers.%d.cross.wo" % i][0].float()[:, :m]      # W^T [out][in]
                want_at = torch.zeros(cfg.heads, J, m, device=cuda)
                want_bt = torch.zeros(m, cfg.heads, J, device=cuda)
                for h in range(cfg.heads):
                    cols = slice(h * hd, (h + 1) * hd)
                    want_at[h, :nc] = d.scale * kv[:, cols] @ wq[:, cols].t()
                    want_bt[:, h, :nc] = wo_t[:, cols] @ kv[:, m:][:, cols].t()
                assert rel(at[i].cpu(), want_at.reshape(-1, m).cpu()) < 5e-3
                assert rel(bt[i].cpu(), want_bt.reshape(m, -1).cpu()) < 5e-3
    assert rel(outs[0], outs[1]) < 5e-3
    assert np.array_equal(outs[0], outs[2])     # the K-band skip only drops exact zero products
    ref = WO.denoise(store.bf16_rounded().params, ocfg, x["motion"], x["z"], x["ref"], x["audio"],
                     np.where(np.arange(Lc) < Lm, 0.0, 0.75))
    assert rel(outs[0], ref) < BUDGET


def test_forward_accepts_any_composite(cuda):
    """Denoiser.forward takes any CompositeInput, like the reference's (net.py:223-238): a
    mask / conditioning layout other than composite_from_state's is patchified as given."""
    from paper_2512_23379_b200.diffusion import composite_from_state
    from paper_2512_23379_b200.net import Denoiser
    cfg, store = _store("default")
    r = np.random.default_rng(4)
    comp = composite_from_state(r.standard_normal((2, 8)), r.standard_normal((7, 8)), r.standard_normal(8),
                                r.uniform(-1, 1, 9), 0.5)
    comp.z_mask[1] = 1.0                       # a second "given" frame
    comp.z_cond[3] = r.standard_normal(8)      # conditioning on another row
    out = Denoiser(cfg).forward(store, comp)
    P = store.bf16_rounded().params
    ref = FO.denoise(P, dict(model_dim=cfg.model_dim, layers=cfg.layers, heads=cfg.heads),
                     {"stacked": comp.stacked(), "frame_t": comp.frame_t, "signal": comp.signal,
                      "reference": comp.reference, "motion_len": comp.motion_len})
    assert rel(out, ref) < 5e-3
    canon = Denoiser(cfg).forward(store, composite_from_state(comp.z_noise[:2], comp.z_noise[2:], comp.reference,
                                                              comp.signal, 0.5))
    assert rel(out, canon) > 1e-3               # the extra mask / cond rows were really used
