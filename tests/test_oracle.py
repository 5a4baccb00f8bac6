"""Pin the CPU oracle to the reference's own outputs (frozen golden vectors).

The golden file is produced by running the reference itself
(`tests/golden/make_golden.py`); tolerance is the reference's backend-parity
tolerance 1e-12 (`pkg/tests/test_backends.py:17`). Integer geometry
(windows, emitted indices) must be exact.
"""

import hashlib

import numpy as np
import pytest

from oracle import ftlk_oracle as O

TOL = dict(rtol=1e-12, atol=1e-12)
CFGS = {"default": (dict(model_dim=32, layers=2, heads=2), 32, 2, 64, 8, 200),
        "tiny": (dict(model_dim=8, layers=1, heads=2), 8, 1, 16, 4, 0),
        "h4": (dict(model_dim=32, layers=2, heads=4), 32, 2, 48, 8, 7)}


def _params(name):
    cfg, m, layers, ff, d, seed = CFGS[name]
    return cfg, O.init_params(O.ftlk_shapes(m, layers, ff, d), seed)


def _checksum(P):
    h = hashlib.sha256()
    for k, v in P.items():
        h.update(k.encode())
        h.update(np.ascontiguousarray(v, dtype=np.float64).tobytes())
    return h.hexdigest()


def test_golden_provenance(golden):
    assert str(golden["backend"]) == "python"
    assert str(golden["numpy_version"]).split(".")[0] == np.__version__.split(".")[0]


def test_kernels_pinned(golden):
    g = golden
    assert np.allclose(O.dense(g["k_dense_x"], g["k_dense_w"], g["k_dense_b"]), g["k_dense_y"], **TOL)
    assert np.allclose(O.gelu(g["k_gelu_x"]), g["k_gelu_y"], **TOL)
    y, mu, rs = O.layernorm(g["k_ln_x"], g["k_ln_g"], g["k_ln_b"])
    for a, b in ((y, "k_ln_y"), (mu, "k_ln_mean"), (rs, "k_ln_rstd")):
        assert np.allclose(a, g[b], **TOL)


@pytest.mark.parametrize("heads", [1, 2, 4])
@pytest.mark.parametrize("cross", [0, 1])
def test_mha_pinned(golden, heads, cross):
    k = "k_mha_h%d_c%d_" % (heads, cross)
    y, cache = O.mha(golden[k + "xq"], golden[k + "xkv"], golden[k + "wq"], golden[k + "wk"],
                     golden[k + "wv"], golden[k + "wo"], heads)
    assert np.allclose(y, golden[k + "y"], **TOL)
    assert np.allclose(cache[3], golden[k + "p"], **TOL)


@pytest.mark.parametrize("name", list(CFGS))
def test_param_init_bit_exact(golden, name):
    _, P = _params(name)
    assert _checksum(P) == str(golden["p_%s_checksum" % name])
    assert sum(v.size for v in P.values()) == int(golden["p_%s_n" % name])


@pytest.mark.parametrize("name", list(CFGS))
@pytest.mark.parametrize("lm", [2, 0, 3])
def test_denoiser_pinned(golden, name, lm):
    cfg, P = _params(name)
    k = "f_%s_lm%d_" % (name, lm)
    comp = O.composite(golden[k + "motion"], golden[k + "z"], golden[k + "ref"],
                       golden[k + "sig"], float(golden[k + "t"]))
    assert np.array_equal(comp["stacked"], golden[k + "stacked"])
    assert np.array_equal(comp["frame_t"], golden[k + "frame_t"])
    assert np.allclose(O.denoise(P, cfg, comp), golden[k + "out"], **TOL)


@pytest.mark.parametrize("steps", [4, 2, 1])
def test_sampler_pinned(golden, steps):
    cfg, P = _params("default")
    k = "s_steps%d_" % steps
    tr = []
    lat = O.sample_chunk(lambda c: O.denoise(P, cfg, c), golden[k + "timesteps"], golden["s_motion"],
                         golden["s_ref"], golden["s_sig"], rng=O.rng_for(5, O.STREAM_NOISE, 3), trace=tr)
    assert np.allclose(lat, golden[k + "latents"], **TOL)
    assert np.allclose(np.stack([t[1] for t in tr]), golden[k + "z"], **TOL)
    assert np.allclose(np.stack([t[2] for t in tr]), golden[k + "x0"], **TOL)


def test_rollout_and_decode_pinned(golden):
    cfg, P = _params("default")
    targets, motions, idx = O.rollout(lambda c: O.denoise(P, cfg, c), (1.0, 0.75, 0.5, 0.25),
                                      golden["r_reference_latent"], golden["r_signal"], 35,
                                      int(golden["r_seed"]))
    assert np.allclose(targets, golden["r_targets"], **TOL)
    assert np.allclose(np.stack(motions), golden["r_motions"], **TOL)
    assert np.allclose(O.codec_decode(targets, golden["r_Q"]), golden["r_frames"], **TOL)
    # engine twin: the threaded reference engine emitted the same indices/states
    assert np.array_equal(idx, golden["e_index"])
    assert np.array_equal(idx // 7, golden["e_chunk"])
    assert np.allclose(O.codec_decode(targets, golden["r_Q"]), golden["e_state"], **TOL)
    assert np.allclose(O.codec_encode(golden["r_reference_frame"][None], golden["r_Q"])[0],
                       golden["r_reference_latent"], **TOL)


@pytest.mark.parametrize("lc,lm", [(9, 2), (5, 0), (6, 5)])
def test_windows_exact(golden, lc, lm):
    wins = np.stack([O.window(golden["w_signal"], c, lc, lm) for c in range(4)])
    assert np.array_equal(wins, golden["w_%d_%d" % (lc, lm)])


@pytest.mark.parametrize("name", list(CFGS))
def test_product_param_init_matches_reference(golden, name):
    """The product ParamStore.init reproduces the reference init bit for bit."""
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    _, m, layers, ff, d, seed = CFGS[name]
    heads = CFGS[name][0]["heads"]
    st = ParamStore.init(NetConfig(m, layers, heads, ff, d), seed)
    assert st.checksum() == str(golden["p_%s_checksum" % name])


@pytest.mark.parametrize("steps", [4, 2, 1])
def test_product_chunk_noise_bit_exact(golden, steps):
    """Initial sampler noise: the product's host draw is the reference's draw."""
    from paper_2512_23379_b200.seeding import chunk_noise
    z = chunk_noise(5, 3, golden["s_steps%d_z" % steps][0].shape)
    assert np.array_equal(z, golden["s_steps%d_z" % steps][0])


def test_rope_tables_bit_exact():
    """Product RoPE tables (host float64 -> float32) equal the oracle's, byte for byte,
    and the per-token expansion is an exact gather of them."""
    from oracle import wan_oracle as WO
    from paper_2512_23379_b200.rope import per_token_tables, rope3d_tables
    for hd, F, gh, gw in [(128, 10, 26, 45), (64, 4, 6, 9), (16, 3, 2, 2)]:
        a, b = rope3d_tables(F, gh, gw, hd), WO.rope_tables(F, gh, gw, hd)
        for k in a:
            assert a[k].dtype == np.float32 and a[k].tobytes() == b[k].tobytes(), (hd, k)
        cos, sin = per_token_tables(a, gh, gw)
        assert cos.shape == (F * gh * gw, hd // 2)
        r, c = min(5, gh - 1), min(3, gw - 1)
        t = gh * gw + r * gw + c  # frame 1, row r, col c
        assert np.array_equal(cos[t], np.concatenate([a["cos_t"][1], a["cos_h"][r], a["cos_w"][c]]))
        assert np.array_equal(sin[t], np.concatenate([a["sin_t"][1], a["sin_h"][r], a["sin_w"][c]]))
