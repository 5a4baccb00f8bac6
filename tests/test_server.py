"""WebSocket front door (reference tests/test_server.py protocol cases) over the
B200 engine. Message-validation cases never open a session and run on CPU; the
frame-flow case needs the device engine (gpu marker)."""

import json
import types

import numpy as np
import pytest

pytest.importorskip("fastapi")
from starlette.testclient import TestClient  # noqa: E402


class _World:
    """Duck-typed reference World built from the frozen readouts (world.py:76-120)."""

    def __init__(self, golden):
        self.P = golden["r_P"]
        self.w = golden["r_w"]
        self.spec = types.SimpleNamespace(identity_dim=self.P.shape[1])

    def mouth(self, frames):
        return np.asarray(frames, dtype=np.float64) @ self.w


@pytest.fixture(scope="module")
def app(golden):
    from paper_2512_23379_b200.codec import Codec
    from paper_2512_23379_b200.config import NetConfig
    from paper_2512_23379_b200.net import ParamStore
    from paper_2512_23379_b200.server import build_app
    cfg = NetConfig()
    return build_app(ParamStore.init(cfg, 200), cfg, _World(golden), Codec(golden["r_Q"]), pacing="unpaced")


@pytest.fixture()
def ws(app):
    from paper_2512_23379_b200.server import WS_PATH
    with TestClient(app).websocket_connect(WS_PATH) as sock:
        yield sock


def _recv(sock):
    return json.loads(sock.receive_text())


def _send(sock, **msg):
    sock.send_text(json.dumps(msg))


def test_drive_before_start_errors(ws):
    _send(ws, type="drive", index=0, value=0.1)
    m = _recv(ws)
    assert m["type"] == "error" and "before start" in m["message"]


def test_invalid_json_errors(ws):
    ws.send_text("{not json")
    assert _recv(ws) == {"type": "error", "message": "message is not valid JSON"}
    _send(ws, type="drive", index=0, value=0.0)   # socket still usable
    assert _recv(ws)["type"] == "error"


def test_unknown_type_errors(ws):
    _send(ws, type="dance")
    m = _recv(ws)
    assert m["type"] == "error" and "unknown message type" in m["message"]


def test_bad_identity_errors(ws, golden):
    for ident in ([1.0], [0.0] * golden["r_P"].shape[1], [float("nan")] * golden["r_P"].shape[1]):
        _send(ws, type="start", seed=1, identity=ident)
        m = _recv(ws)
        assert m["type"] == "error" and m["message"].startswith("bad start message"), m


def test_bad_start_fields_error(ws):
    _send(ws, type="start", identity=[1.0, 0.0])
    assert _recv(ws)["message"].startswith("bad start message")


def test_stop_without_start_is_clean(ws):
    _send(ws, type="stop")


@pytest.mark.gpu
def test_frames_flow_in_order_and_match_engine(ws, golden, cuda):
    """35 drive samples -> frames 0..34 in order with chunk = index // 7, a stats message
    after every chunk; states equal a direct StreamSession fed the same reference frame
    (P @ normalised identity), mouth = state @ w."""
    from paper_2512_23379_b200.codec import Codec
    from paper_2512_23379_b200.config import NetConfig, StreamConfig
    from paper_2512_23379_b200.net import ParamStore
    from paper_2512_23379_b200.streaming import start_stream
    ident = golden["r_identity"] * 3.0          # server normalises
    sig = golden["r_signal"][:35]
    _send(ws, type="start", seed=11, identity=list(ident), fps=25.0)
    for j, v in enumerate(sig):
        _send(ws, type="drive", index=j, value=float(v))
    frames, stats = [], []
    while len(frames) < 35 or len(stats) < 5:
        m = _recv(ws)
        assert m["type"] in ("frame", "stats"), m
        (frames if m["type"] == "frame" else stats).append(m)
    assert [f["index"] for f in frames] == list(range(35))
    assert [f["chunk"] for f in frames] == [i // 7 for i in range(35)]
    assert set(stats[-1]) == {"type", "startup_ms", "fps", "cycle"} and stats[-1]["fps"] > 0
    _send(ws, type="stop")
    cfg = NetConfig()
    sess = start_stream(ParamStore.init(cfg, 200), cfg, Codec(golden["r_Q"]),
                        golden["r_P"] @ (ident / np.linalg.norm(ident)), StreamConfig(seed=11))
    sess.push_signal((j, float(v)) for j, v in enumerate(sig))
    direct = []
    while len(direct) < 35:
        fr, _ = sess.next_frames(wait=True, timeout=0.5)
        direct.extend(fr)
    sess.close()
    want = np.stack([f.state for f in direct])
    got = np.array([f["state"] for f in frames])
    assert np.array_equal(got, want)
    assert np.allclose([f["mouth"] for f in frames], want @ golden["r_w"], rtol=0, atol=1e-12)
