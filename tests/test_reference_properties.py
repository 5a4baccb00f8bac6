"""Behavioural properties the reference's own tests pin for this path,
restated against this package: sampler exactness with an oracle / zero denoiser
(`tests/test_diffusion.py:126-154`), composite layout (`:42-62`), codec round trip
(`tests/test_world.py:99-115`), and on the device: zero params -> zero output,
determinism, intra-chunk bidirectionality (`tests/test_net.py:30-56`), bit-exact
cross-chunk causality and the last window sample reaching the first frame
(`tests/test_streaming.py:132-173`)."""

import numpy as np
import pytest

from paper_2512_23379_b200.config import NetConfig, NoiseSchedule, SamplerPlan, StreamConfig
from paper_2512_23379_b200.diffusion import composite_from_state, few_step_sample

PLANS = [SamplerPlan(steps=1, timesteps=(1.0,)), SamplerPlan(steps=2, timesteps=(1.0, 0.5)),
         SamplerPlan(steps=4, timesteps=(1.0, 0.75, 0.5, 0.25))]


@pytest.mark.parametrize("plan", PLANS)
def test_sampler_with_oracle_denoiser_returns_ground_truth(plan):
    r = np.random.default_rng(6)
    lm, lc, d = 2, 9, 4
    gt = r.standard_normal((lc, d))
    chunk = few_step_sample(lambda comp: gt.copy(), plan, gt[:lm], r.standard_normal(d), r.standard_normal(lc),
                            np.random.default_rng(0))
    assert np.max(np.abs(chunk.latents[lm:] - gt[lm:])) < 1e-9
    assert np.array_equal(chunk.latents[:lm], gt[:lm])


def test_sampler_with_zero_denoiser_rescales_by_sigma_ratio():
    plan = SamplerPlan(steps=3, timesteps=(1.0, 0.6, 0.3))
    sched = NoiseSchedule()
    lm, lc, d = 1, 6, 3
    trace = []
    chunk = few_step_sample(lambda comp: np.zeros((lc, d)), plan, np.zeros((lm, d)), np.zeros(d), np.zeros(lc),
                            np.random.default_rng(1), trace=trace)
    assert np.all(chunk.latents[lm:] == 0.0)
    for (ta, za, _), (tb, zb, _) in zip(trace, trace[1:]):
        assert np.allclose(zb, za * sched.sigma(tb) / sched.sigma(ta), atol=1e-12)


def test_composite_layout():
    r = np.random.default_rng(2)
    motion, z, ref, sig = r.standard_normal((2, 8)), r.standard_normal((7, 8)), r.standard_normal(8), r.uniform(-1, 1, 9)
    comp = composite_from_state(motion, z, ref, sig, 0.75)
    st = comp.stacked()
    assert st.shape == (9, 17)
    assert np.array_equal(st[:, :8], np.concatenate([motion, z]))             # z_noise = [motion; z]
    assert np.array_equal(st[:, 8], np.eye(9)[0])                              # z_mask = [1, 0, ...]
    assert np.array_equal(st[0, 9:], ref) and np.all(st[1:, 9:] == 0)         # z_cond row 0 = reference
    assert np.array_equal(comp.frame_t, [0.0, 0.0] + [0.75] * 7)               # motion rows at t = 0


def test_codec_round_trip(golden):
    from paper_2512_23379_b200.codec import Codec
    codec = Codec(golden["r_Q"])
    x = np.random.default_rng(3).standard_normal((11, golden["r_Q"].shape[0]))
    assert np.max(np.abs(codec.decode(codec.encode(x)) - x)) < 1e-12


# ---------------------------------------------------------------- device properties
def _comp(r, cfg, lm=2, lc=9, t=0.6):
    d = cfg.latent_dim
    return composite_from_state(r.standard_normal((lm, d)), r.standard_normal((lc - lm, d)), r.standard_normal(d),
                                r.uniform(-1, 1, lc), t)


@pytest.mark.gpu
def test_zero_params_zero_output(cuda):
    from paper_2512_23379_b200.net import Denoiser, ParamStore
    cfg = NetConfig()
    out = Denoiser(cfg).forward(ParamStore.zeros(cfg), _comp(np.random.default_rng(0), cfg))
    assert np.all(out == 0.0)


@pytest.mark.gpu
def test_forward_deterministic(cuda):
    from paper_2512_23379_b200.net import Denoiser
    cfg = NetConfig()
    net = Denoiser(cfg)
    store = net.init_params(3)
    comp = _comp(np.random.default_rng(1), cfg)
    assert np.array_equal(net.forward(store, comp), net.forward(store, comp))


@pytest.mark.gpu
def test_future_frames_influence_past_predictions(cuda):
    from paper_2512_23379_b200.net import Denoiser
    cfg = NetConfig()
    net = Denoiser(cfg)
    store = net.init_params(4)
    comp = _comp(np.random.default_rng(2), cfg, lm=1, lc=6, t=0.4)
    swapped = composite_from_state(comp.z_noise[:1], comp.z_noise[1:][[0, 1, 3, 2, 4]], comp.z_cond[0], comp.signal,
                                   0.4)
    a, b = net.forward(store, comp), net.forward(store, swapped)
    assert not np.allclose(a[1], b[1])


def _session_frames(golden, sig, n, seed):
    from paper_2512_23379_b200.codec import Codec
    from paper_2512_23379_b200.net import ParamStore
    from paper_2512_23379_b200.streaming import start_stream
    cfg = NetConfig()
    sess = start_stream(ParamStore.init(cfg, 200), cfg, Codec(golden["r_Q"]), golden["r_reference_frame"],
                        StreamConfig(seed=seed))
    sess.push_signal(list(enumerate(sig)))
    got = []
    while len(got) < n:
        fr, _ = sess.next_frames(wait=True, timeout=0.5)
        got.extend(fr)
    sess.close()
    return got


@pytest.mark.gpu
def test_future_samples_do_not_change_past_chunks(golden, cuda):
    sig = np.asarray(golden["r_signal"][:28], dtype=np.float64)
    bent = sig.copy()
    bent[14:] = np.clip(bent[14:] + 0.25, -1, 1)
    a = _session_frames(golden, sig, 28, 4)
    b = _session_frames(golden, bent, 28, 4)
    for x, y in zip(a[:14], b[:14]):                          # chunks 0-1: bit-identical
        assert x.index == y.index and np.array_equal(x.state, y.state)
    assert any(not np.array_equal(x.state, y.state) for x, y in zip(a[14:], b[14:]))


@pytest.mark.gpu
def test_last_sample_in_window_matters(golden, cuda):
    sig = np.asarray(golden["r_signal"][:7], dtype=np.float64)
    hi, lo = sig.copy(), sig.copy()
    hi[-1], lo[-1] = 0.9, -0.9
    a = _session_frames(golden, hi, 7, 5)
    b = _session_frames(golden, lo, 7, 5)
    assert not np.allclose(a[0].state, b[0].state)
