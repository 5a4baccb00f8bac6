"""Parity at the production widths and token counts ("re-measure at L = 10 530"),
in the driver-run `-m gpu` suite.

* DiT at the 14B width (m 5120 / 40 heads / ff 13 824) and the 1.3B width (1536 / 12 / 8 960),
  full streaming geometry 416x720 -> L = 9 x 1170 = 10 530 tokens, 2 layers: one 4-step chunk
  through the public sampler API (`few_step_sample` over `Denoiser.as_denoise_fn`, the
  reference's `diffusion.py:202-237` / `net.py:371-375` boundary) against the fp64 oracle
  (`oracle/wan_oracle.sample_chunk`) with shared bf16-rounded weights. Every step's x0
  prediction is compared (step 0 is a plain forward at t = 1) and the chunk's targets.
* The causal VAE decoder at the production widths (base 96: 384/384/384/192/96, 3 res blocks
  per level, temporal x2 at the first two upsamples) on a cropped latent grid, two chunks (the
  second runs on the causal caches of the first), float and RGB8 outputs, against
  `oracle/vae_oracle.VAEOracle`.

Bar: relative L2 <= 1e-2 (north star). Values are printed in the pytest terminal summary.
"""

import numpy as np
import pytest
import torch

from oracle import vae_oracle as VO
from oracle import wan_oracle as WO

pytestmark = pytest.mark.gpu
BUDGET = 1e-2

WIDTHS = {"14b": (5120, 40, 13824), "1.3b": (1536, 12, 8960)}


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("width", ["1.3b", "14b"])
def test_wan_width_full_tokens_chunk(cuda, record_parity, width):
    from paper_2512_23379_b200.config import NetConfig, SamplerPlan
    from paper_2512_23379_b200.diffusion import few_step_sample
    from paper_2512_23379_b200.net import Denoiser, ParamStore
    from paper_2512_23379_b200.seeding import STREAM_NOISE, rng_for
    m, heads, ff = WIDTHS[width]
    layers, D, A, adim, Lc, Lm, H, W = 2, 16, 4, 768, 9, 2, 52, 90
    cfg = NetConfig(m, layers, heads, ff, D, mode="wan", patch=(1, 2, 2), audio_dim=adim, audio_tokens=A)
    store = ParamStore.init(cfg, 200)
    for v in store.params.values():      # shared bf16 weights (one host copy, rounded in place)
        v[...] = torch.from_numpy(v).to(torch.bfloat16).to(torch.float64).numpy()
    r = np.random.default_rng(1)
    motion, ref = r.standard_normal((Lm, D, H, W)), r.standard_normal((D, H, W))
    audio = r.standard_normal((Lc, A, adim))
    assert Lc * (H // 2) * (W // 2) == 10530
    plan = SamplerPlan()
    tr = []
    chunk = few_step_sample(Denoiser(cfg).as_denoise_fn(store), plan, motion, ref, audio,
                            rng_for(11, STREAM_NOISE, 0), trace=tr)
    z0 = rng_for(11, STREAM_NOISE, 0).standard_normal((Lc - Lm, D, H, W))
    ocfg = dict(model_dim=m, layers=layers, heads=heads, latent_dim=D, patch=(1, 2, 2), audio_tokens=A,
                audio_dim=adim)
    otr = []
    want = WO.sample_chunk(store.params, ocfg, plan.timesteps, motion, ref, audio, z0, trace=otr)
    assert np.array_equal(chunk.latents[:Lm], motion)            # carried motion rows, exact
    errs = []
    for i, t in enumerate(plan.timesteps):
        e = rel(tr[i][2], otr[i][2])
        record_parity("x0 step %d (t=%.2f)" % (i, t), e)
        errs.append(e)
    ec = rel(chunk.targets, want[Lm:])
    record_parity("chunk targets", ec)
    assert max(errs) < BUDGET and ec < BUDGET, (errs, ec)


WAN_VAE = dict(z_dim=16, base_dim=96, dim_mult=(1, 2, 4, 4), num_res_blocks=2, temporal_upsample=(True, True, False))


def test_vae_production_width_two_chunks(cuda, record_parity):
    """Full-width decoder (the bench's), 7 latent frames of a 4 x 18 crop -> 28 frames of
    32 x 144 px (ragged 128-pixel tiles at full resolution), two chunks."""
    from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig, init_vae_params

    def bfr(x):
        return torch.as_tensor(x).to(torch.bfloat16).to(torch.float64).numpy()
    cfg = VAEConfig(**WAN_VAE)
    assert cfg.dims == [384, 384, 384, 192, 96]
    P = init_vae_params(cfg, 3)
    orc = VO.VAEOracle({k: (bfr(v) if k.endswith(".w") else v) for k, v in P.items()}, **WAN_VAE)
    dec = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=False)
    dec8 = DeviceVAEDecoder(cfg, cuda, params=P, rgb8=True)
    r = np.random.default_rng(2)
    s = torch.cuda.current_stream()
    for c in range(2):
        z = r.standard_normal((7, 16, 4, 18))
        want = orc.decode(z)
        zd = torch.as_tensor(z, dtype=torch.float32, device=cuda)
        got = dec.decode_device(zd, s)[..., :3]
        assert got.shape == want.shape == (28, 32, 144, 3)
        e = rel(got, want)
        record_parity("decode chunk %d" % c, e)
        assert e < BUDGET, (c, e)
        rgb = dec8.decode_device(zd, s)
        d = np.abs(rgb.astype(int) - VO.to_rgb8(want).astype(int))
        record_parity("rgb8 chunk %d frac |d|<=2" % c, float(np.mean(d <= 2)))
        assert rgb.dtype == np.uint8 and rgb.shape == (28, 32, 144, 3)
        assert np.mean(d <= 2) > 0.99
