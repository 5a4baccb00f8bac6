"""FTLK checkpoint I/O against a file written by the reference's own writer
(tests/golden/tiny.ftlk, made by tests/golden/make_golden.py)."""

import os

import numpy as np
import pytest

from paper_2512_23379_b200 import checkpoint as CK
from paper_2512_23379_b200.config import NetConfig
from paper_2512_23379_b200.errors import ConfigError
from paper_2512_23379_b200.net import ParamStore

GOLD = os.path.join(os.path.dirname(__file__), "golden", "tiny.ftlk")


def test_load_reference_checkpoint(golden):
    store, role, net = CK.load(GOLD)
    assert role == "generator_student"
    assert net == NetConfig(8, 1, 2, 16, 4)
    assert store.checksum() == str(golden["c_tiny_checksum"])


def test_save_is_byte_identical_to_reference_writer(tmp_path):
    store, role, net = CK.load(GOLD)
    out = tmp_path / "re.ftlk"
    CK.save(out, store, role, net)
    assert out.read_bytes() == open(GOLD, "rb").read()


def test_wan_roundtrip(tmp_path):
    cfg = NetConfig(64, 1, 2, 128, 4, mode="wan", patch=(1, 2, 2), audio_dim=8, audio_tokens=2)
    st = ParamStore.init(cfg, 3)
    p = tmp_path / "w.ftlk"
    CK.save(p, st, "teacher_real", cfg)
    st2, role, cfg2 = CK.load(p)
    assert cfg2 == cfg and role == "teacher_real" and st2.checksum() == st.checksum()


@pytest.mark.parametrize("mutate", ["magic", "truncate", "trailing", "version"])
def test_strict_errors(tmp_path, mutate):
    blob = bytearray(open(GOLD, "rb").read())
    if mutate == "magic":
        blob[:4] = b"XXXX"
    elif mutate == "truncate":
        blob = blob[:-10]
    elif mutate == "trailing":
        blob += b"\0"
    else:
        blob[4] = 2
    p = tmp_path / "bad.ftlk"
    p.write_bytes(bytes(blob))
    with pytest.raises(ConfigError):
        CK.load(p)


@pytest.mark.gpu
def test_streaming_device_loader(cuda):
    w, role, net = CK.load_device_weights(GOLD, cuda)
    store, _, _ = CK.load(GOLD)
    import torch
    wt, K = w.mats["in.w"]
    assert K == 9 and torch.equal(wt[:, :K].cpu(), torch.from_numpy(store.params["in.w"].T.copy()).to(torch.bfloat16))
    assert np.allclose(w.vecs["final.g"].cpu().numpy(), store.params["final.g"])


@pytest.mark.parametrize("cut", [10, 300, 2000])
def test_device_loader_truncated_raises_config_error(tmp_path, cut):
    """A malformed file reaches the caller as ConfigError, not as the BufferError of closing a
    still-exported mapping (the failure happens in validation, before any device copy)."""
    blob = open(GOLD, "rb").read()
    p = tmp_path / "trunc.ftlk"
    p.write_bytes(blob[:-cut])
    with pytest.raises(ConfigError):
        CK.load_device_weights(p, device="cpu")
