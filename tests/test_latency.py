"""Latency model (reference tests/test_latency.py cases, restated) and the B200
recalibration from bench lines. CPU only."""

import json

import numpy as np
import pytest

from paper_2512_23379_b200 import latency as LT
from paper_2512_23379_b200.errors import ConfigError


def test_single_gpu_pays_no_comm():
    s = LT.PipelineSpec(gpu_count=1)
    assert s.dit_step_ms() == s.dit_step_ms_1gpu and s.vae_decode_ms() == s.vae_decode_ms_1gpu


def test_components_scale_and_comm_floor():
    s = LT.PipelineSpec()
    assert s.dit_step_ms(8) == pytest.approx(1070.0 / 8 + 59.25)
    big = LT.PipelineSpec(gpu_count=8, dit_step_ms_1gpu=1e-9, vae_encode_ms_1gpu=0, vae_decode_ms_1gpu=0)
    r = LT.predict(big)
    assert r.cycle_ms == pytest.approx(33 + 26 + 4 * 59.25 + 8.875 + 68.5, rel=1e-9)


def test_fps_identity_and_monotone():
    prev = None
    for g in (1, 2, 4, 8):
        r = LT.predict(LT.PipelineSpec(gpu_count=g))
        assert r.fps == pytest.approx(28 * 1000.0 / r.cycle_ms)
        if prev is not None:
            assert r.cycle_ms < prev
        prev = r.cycle_ms
    d = LT.predict(LT.PipelineSpec()).to_dict()
    assert LT.LatencyReport(**d).to_dict() == d


def test_calibrate_two_point_and_lstsq():
    f = LT.calibrate([(1, 1070.0), (8, 193.0)])
    assert f["compute_ms_1gpu"] == 1070.0 and f["comm_ms"] == pytest.approx(193.0 - 1070.0 / 8)
    f = LT.calibrate([(2, 600.0), (4, 350.0)])
    assert f["compute_ms_1gpu"] / 2 + f["comm_ms"] == pytest.approx(600.0)
    pts = [(g, 800.0 / g + (12.5 if g > 1 else 0.0)) for g in (1, 2, 4, 8)]
    f = LT.calibrate(pts, base_ms_1gpu=1000.0)
    assert f["compute_ms_1gpu"] == pytest.approx(800.0) and f["comm_ms"] == pytest.approx(12.5)
    assert f["compile_speedup"] == pytest.approx(0.8) and np.allclose(f["residuals"], 0, atol=1e-9)
    with pytest.raises(ConfigError):
        LT.calibrate([(4, 1.0), (4, 2.0)])


def test_calibrate_spec_both_table_forms():
    _, measured = LT.load_bundled_spec("paper_h800")
    tab = {k: {int(g): v for g, v in d.items()} for k, d in measured["table_component_ms"].items()}
    a = LT.calibrate_spec(LT.PipelineSpec(), tab)
    b = LT.calibrate_spec(LT.PipelineSpec(), [(g, k, v) for k, d in tab.items() for g, v in d.items()])
    assert a == b and a.dit_comm_ms == pytest.approx(193.0 - 1070.0 / 8)
    with pytest.raises(ConfigError):
        LT.calibrate_spec(LT.PipelineSpec(), {"dit_step": {1: 1.0, 2: 1.0}})


def test_compose_cycle():
    _, measured = LT.load_bundled_spec()
    c = LT.compose_cycle(measured["cycle_breakdown_8gpu_ms"])
    assert c["cycle_ms"] == 876.0 and c["fps"] == pytest.approx(28000 / 876.0)
    with pytest.raises(ConfigError):
        LT.compose_cycle({"signal_ms": 1.0})


def test_simulate_serial_equals_predict_and_overlap_helps():
    s = LT.PipelineSpec()
    ev, steady = LT.simulate_pipeline(s, 5)
    assert steady == pytest.approx(LT.predict(s).cycle_ms)
    assert len(ev) == 25 and ev[0]["stage"] == "signal"
    _, one = LT.simulate_pipeline(s, 1)
    assert one == pytest.approx(LT.predict(s).cycle_ms)
    _, ov = LT.simulate_pipeline(s, 6, overlap="decode_overlaps_denoise")
    assert ov < steady
    for bad in (dict(n_cycles=0), dict(n_cycles=2, overlap="x")):
        with pytest.raises(ConfigError):
            LT.simulate_pipeline(s, **bad)


def test_spec_validation_and_files(tmp_path):
    with pytest.raises(ConfigError):
        LT.PipelineSpec(gpu_count=0)
    with pytest.raises(ConfigError):
        LT.PipelineSpec(compile_speedup=1.5)
    p = tmp_path / "s.json"
    p.write_text(json.dumps({"spec": {"gpu_count": 2}}))
    assert LT.spec_from_file(p)[0].gpu_count == 2
    p.write_text("{}")
    with pytest.raises(ConfigError):
        LT.spec_from_file(p)


def test_b200_spec_from_bench_lines():
    one = {"n_gpus": 1, "components_ms": {"denoise": 1200.0, "decode": 200.0, "steps_per_chunk": 4,
                                          "frames_per_chunk": 28}}
    s = LT.spec_from_bench([one])
    assert s.dit_step_ms_1gpu == 300.0 and s.vae_decode_ms_1gpu == 200.0 and s.vae_encode_ms_1gpu == 0.0
    eight = {"n_gpus": 8, "components_ms": {"denoise": 1200.0 / 8 + 4 * 10.0, "decode": 200.0 / 8 + 5.0}}
    s8 = LT.spec_from_bench([one, eight])
    assert s8.dit_comm_ms == pytest.approx(10.0) and s8.vae_decode_comm_ms == pytest.approx(5.0)
    with pytest.raises(ConfigError):
        LT.spec_from_bench([eight])


def test_bundled_b200_spec_is_consistent():
    s, measured = LT.load_bundled_spec("paper_b200")
    assert s.vae_encode_ms_1gpu == 0.0 and s.denoise_steps == 4
    line = measured["bench_line_1gpu"]
    r = LT.predict(LT.PipelineSpec(**{**s.__dict__, "gpu_count": 1, "audio_ms": 0.0, "misc_ms": 0.0}))
    assert r.cycle_ms == pytest.approx(line["components_ms"]["denoise"] + line["components_ms"]["decode"])
