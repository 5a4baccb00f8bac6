"""Streaming engine on the B200 against the reference's recorded rollout and
threaded-engine outputs (golden vectors), plus the engine contracts the
reference tests (ordering, replay, cold start, flat memory, input errors)."""

import time

import numpy as np
import pytest

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


def test_generate_free_running_drift(golden, cuda, setup):
    from paper_2512_23379_b200.config import StreamConfig
    from paper_2512_23379_b200.streaming import generate
    cfg, store, codec = setup
    tg, _, frames = generate(store, cfg, codec, golden["r_reference_latent"], golden["r_signal"], 35,
                             cfg=StreamConfig(seed=int(golden["r_seed"])))
    drift = [rel(tg[7 * c:7 * c + 7], golden["r_targets"][7 * c:7 * c + 7]) for c in range(5)]
    print("free-running per-chunk rel-L2:", ["%.2e" % d for d in drift])
    assert drift[0] < BUDGET
    assert max(drift) < 5 * BUDGET


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
