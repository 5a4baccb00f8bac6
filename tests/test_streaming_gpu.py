"""Streaming engine on the B200 against the reference's recorded rollout and
threaded-engine outputs (golden vectors), plus the engine contracts the
reference tests (ordering, replay, cold start, flat memory, input errors)."""

import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
BUDGET = 1e-2


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def setup(golden):
    from paper_2512_23379_b200.codec import Codec
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    cfg = NetConfig()
    return cfg, ParamStore.init(cfg, 200), Codec(golden["r_Q"])


def test_generate_teacher_forced_per_chunk(golden, cuda, setup):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import generate
    cfg, store, codec = setup
    scfg = StreamConfig(seed=int(golden["r_seed"]))
    tg, motions, frames = generate(store, cfg, codec, golden["r_reference_latent"], golden["r_signal"], 35,
                                   cfg=scfg, motion_override=golden["r_motions"])
    for c in range(5):
        assert rel(tg[7 * c:7 * c + 7], golden["r_targets"][7 * c:7 * c + 7]) < BUDGET, c
    assert rel(frames, golden["r_frames"]) < BUDGET
    # cold start: chunk 0 conditions on L_m copies of the encoded reference
    assert np.allclose(motions[0], np.repeat(golden["r_reference_latent"][None], 2, 0), atol=1e-6)


def test_generate_free_running_drift(golden, cuda, setup, record_parity):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import generate
    cfg, store, codec = setup
    tg, _, frames = generate(store, cfg, codec, golden["r_reference_latent"], golden["r_signal"], 35,
                             cfg=StreamConfig(seed=int(golden["r_seed"])))
    drift = [rel(tg[7 * c:7 * c + 7], golden["r_targets"][7 * c:7 * c + 7]) for c in range(5)]
    for c, d in enumerate(drift):
        record_parity("free-running chunk %d" % c, d)
    assert max(drift) < BUDGET   # the north-star budget holds across the whole 5-chunk rollout


def _run_session(store, cfg, codec, golden, n=35, push_in=(35,)):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import start_stream
    sess = start_stream(store, cfg, codec, golden["r_reference_frame"], StreamConfig(seed=int(golden["r_seed"])))
    got = []
    fed = 0
    for upto in push_in:
        sess.push_signal((i, golden["r_signal"][i]) for i in range(fed, upto))
        fed = upto
    deadline = time.time() + 120
    while len(got) < n and time.time() < deadline:
        fr, _ = sess.next_frames(wait=True, timeout=0.2)
        got.extend(fr)
    stats = sess.stats()
    sess.close()
    return got, stats


def test_session_matches_reference_engine(golden, cuda, setup):
    cfg, store, codec = setup
    got, stats = _run_session(store, cfg, codec, golden, push_in=(3, 10, 20, 35))
    assert [f.index for f in got] == list(golden["e_index"])          # bit-exact ordering / indices
    assert [f.chunk for f in got] == list(golden["e_chunk"])
    states = np.stack([f.state for f in got])
    assert rel(states[:7], golden["e_state"][:7]) < BUDGET
    assert stats.frames_emitted == 35 and stats.chunks_emitted == 5
    # the threaded engine and the synchronous twin are the same computation
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import generate
    _, _, fr = generate(store, cfg, codec, golden["r_reference_latent"], golden["r_signal"], 35,
                        cfg=StreamConfig(seed=int(golden["r_seed"])))
    assert np.array_equal(states, fr)


def test_session_replay_bit_identical(golden, cuda, setup):
    cfg, store, codec = setup
    a, _ = _run_session(store, cfg, codec, golden)
    b, _ = _run_session(store, cfg, codec, golden, push_in=(7, 35))
    assert np.array_equal(np.stack([f.state for f in a]), np.stack([f.state for f in b]))


def test_session_input_contract(golden, cuda, setup):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.errors import ConfigError
    from paper_2512_23379_b200.streaming import start_stream
    cfg, store, codec = setup
    sess = start_stream(store, cfg, codec, golden["r_reference_frame"], StreamConfig())
    with pytest.raises(ConfigError):
        sess.push_signal([(1, 0.0)])
    with pytest.raises(ConfigError):
        sess.push_signal([(0, float("nan"))])
    sess.close()
    with pytest.raises(ConfigError):
        sess.push_signal([(0, 0.0)])


def test_session_memory_flat(golden, cuda, setup):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import start_stream
    cfg, store, codec = setup
    sess = start_stream(store, cfg, codec, golden["r_reference_frame"], StreamConfig(seed=1))
    sig = np.sin(np.arange(7 * 60) / 5.0)
    marks = {}
    fed, got = 0, 0
    deadline = time.time() + 300
    while got < len(sig) and time.time() < deadline:
        if fed < min(len(sig), got + 21):
            up = min(len(sig), got + 21)
            sess.push_signal((i, sig[i]) for i in range(fed, up))
            fed = up
        fr, _ = sess.next_frames(wait=True, timeout=0.2)
        got += len(fr)
        for f in fr:
            if f.chunk + 1 in (10, 60) and f.index % 7 == 6:
                marks[f.chunk + 1] = sess.persistent_state_nbytes()
    sess.close()
    assert got == len(sig)
    assert marks[60] <= marks[10] * 1.02, marks


def test_wan_stream_with_vae_decoder(cuda):
    """Wan-shaped engine end to end: threaded session with the causal VAE as codec;
    emitted RGB8 frames equal the synchronous twin; decoded float frames of chunk 0
    match the float64 oracle pipeline (DiT sampler -> VAE decode)."""
    from oracle import vae_oracle as VO
    from oracle import wan_oracle as WO
    from paper_2512_23379_b200.config import NetConfig, StreamConfig
    from paper_2512_23379_b200.net import ParamStore
    from paper_2512_23379_b200.seeding import chunk_noise
    from paper_2512_23379_b200.streaming import generate, start_stream
    from paper_2512_23379_b200.vae import DeviceVAEDecoder, VAEConfig, init_vae_params
    cfg = NetConfig(128, 1, 2, 256, 16, mode="wan", patch=(1, 2, 2), audio_dim=8, audio_tokens=2)
    store = ParamStore.init(cfg, 5)
    vcfg = dict(z_dim=16, base_dim=32, dim_mult=(1, 2, 4, 4), num_res_blocks=1, temporal_upsample=(True, True, False))
    VP = init_vae_params(VAEConfig(**vcfg), 6)
    r = np.random.default_rng(2)
    H, W = 4, 6
    ref_lat = r.standard_normal((16, H, W))
    audio = r.standard_normal((14, 2, 8))
    scfg = StreamConfig(chunk_len=5, motion_len=1, seed=9)
    # threaded session, RGB8 output
    vae8 = DeviceVAEDecoder(VAEConfig(**vcfg), cuda, params=VP, rgb8=True)
    sess = start_stream(store, cfg, vae8, None, scfg, reference_latent=ref_lat, latent_hw=(H, W))
    sess.push_signal((i, audio[i]) for i in range(8))
    got = []
    deadline = time.time() + 120
    while len(got) < 32 and time.time() < deadline:
        fr, _ = sess.next_frames(wait=True, timeout=0.2)
        got.extend(fr)
    sess.close()
    assert [f.index for f in got] == list(range(32)) and [f.chunk for f in got] == [i // 16 for i in range(32)]
    assert got[0].state.shape == (32, 48, 3) and got[0].state.dtype == np.uint8
    vae8b = DeviceVAEDecoder(VAEConfig(**vcfg), cuda, params=VP, rgb8=True)
    _, _, fr = generate(store, cfg, vae8b, ref_lat, audio[:8], 8, cfg=scfg, latent_hw=(H, W))
    assert np.array_equal(np.stack([f.state for f in got]), fr)
    # float frames of chunk 0 vs the oracle pipeline
    vaef = DeviceVAEDecoder(VAEConfig(**vcfg), cuda, params=VP, rgb8=False)
    tg, _, frf = generate(store, cfg, vaef, ref_lat, audio[:4], 4, cfg=scfg, latent_hw=(H, W))
    P = store.bf16_rounded().params
    ocfg = dict(model_dim=128, layers=1, heads=2, latent_dim=16, patch=(1, 2, 2), audio_tokens=2, audio_dim=8)
    win = np.concatenate([np.zeros((1, 2, 8)), audio[:4]], 0)
    lat = WO.sample_chunk(P, ocfg, (1.0, 0.75, 0.5, 0.25), ref_lat[None], ref_lat, win,
                          chunk_noise(9, 0, (4, 16, H, W)))
    assert rel(tg[:4], lat[1:]) < BUDGET
    VPb = {k: (torch.as_tensor(v).to(torch.bfloat16).double().numpy() if k.endswith(".w") else v) for k, v in VP.items()}
    want = VO.VAEOracle(VPb, **vcfg).decode(tg[:4])
    assert rel(frf[..., :3], want) < BUDGET


def test_nonfinite_chunk_raises_numeric_error(golden, cuda, setup):
    """A NaN on the numeric path surfaces as the reference's NumericError (errors.py:17-18),
    from generate() and from the live session (device count inside the captured chunk)."""
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.errors import NumericError
    from paper_2512_23379_b200.streaming import generate, start_stream
    cfg, store, codec = setup
    bad = store.clone()
    bad.params["out.b"][3] = np.nan
    with pytest.raises(NumericError):
        generate(bad, cfg, codec, golden["r_reference_latent"], golden["r_signal"], 14,
                 cfg=StreamConfig(seed=int(golden["r_seed"])))
    sess = start_stream(bad, cfg, codec, golden["r_reference_frame"], StreamConfig(seed=int(golden["r_seed"])))
    sess.push_signal((i, golden["r_signal"][i]) for i in range(14))
    with pytest.raises(NumericError):
        deadline = time.time() + 60
        while time.time() < deadline:
            sess.next_frames(wait=True, timeout=0.2)
    sess.close()
