"""Host-side pieces of the front end that need no GPU: the JSON config
schema (config.py, /root/reference/pkg/src/ptychokit/config.py:20-109) and
the 16-bit PNG renders (render.py:25-53), restating the reference's
test_metrics_render.py render assertions."""

import json

import numpy as np
import pytest

from paper_2205_04295_b200 import config as pc
from paper_2205_04295_b200.errors import ParameterError
from paper_2205_04295_b200.render import load_render, plot_error_trace, plot_positions, render


def test_config_merge_defaults_and_overrides(tmp_path, monkeypatch):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"iterations": 3, "posref": {"enabled": True, "kappa": 10}}))
    monkeypatch.delenv(pc.OUTPUT_ENV_VAR, raising=False)
    cfg = pc.load_config(p, pc.RECONSTRUCT_DEFAULTS)
    assert cfg["iterations"] == 3 and cfg["posref"]["kappa"] == 10 and cfg["posref"]["sensor"] == "XCORR_A"
    assert cfg["alpha_object"] == 0.9 and cfg["output_dir"] == "recon"
    monkeypatch.setenv(pc.OUTPUT_ENV_VAR, str(tmp_path / "elsewhere"))
    assert pc.load_config(p, pc.RECONSTRUCT_DEFAULTS)["output_dir"] == str(tmp_path / "elsewhere")
    assert pc.RECONSTRUCT_DEFAULTS["iterations"] == 100          # defaults untouched


@pytest.mark.parametrize("payload,msg", [({"sede": 1}, "sede"), ({"posref": {"kapa": 3}}, "posref.kapa")])
def test_config_unknown_keys_rejected(tmp_path, payload, msg):
    p = tmp_path / "c.json"
    p.write_text(json.dumps(payload))
    with pytest.raises(ParameterError, match=msg):
        pc.load_config(p, pc.RECONSTRUCT_DEFAULTS)


def test_config_bad_files(tmp_path):
    with pytest.raises(ParameterError):
        pc.load_config(tmp_path / "missing.json", pc.SIMULATE_DEFAULTS)
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(ParameterError):
        pc.load_config(tmp_path / "bad.json", pc.SIMULATE_DEFAULTS)
    (tmp_path / "list.json").write_text("[1, 2]")
    with pytest.raises(ParameterError):
        pc.load_config(tmp_path / "list.json", pc.SIMULATE_DEFAULTS)


def test_render_magnitude_round_trip_within_quantization(tmp_path):
    f = np.random.default_rng(0).standard_normal((16, 16)) * (1 + 1j)
    values, sidecar = load_render(render(f, "magnitude", tmp_path / "m.png"))
    span = sidecar["vmax"] - sidecar["vmin"]
    assert np.max(np.abs(values - np.abs(f))) <= span / 65535 + 1e-12
    assert sidecar["kind"] == "magnitude" and sidecar["shape"] == [16, 16]


def test_render_phase_scale_fixed(tmp_path):
    f = np.exp(1j * np.linspace(-3, 3, 64)).reshape(8, 8)
    values, sidecar = load_render(render(f, "phase", tmp_path / "p.png"))
    assert sidecar["vmin"] == -np.pi and sidecar["vmax"] == np.pi
    assert np.max(np.abs(values - np.angle(f))) <= 2 * np.pi / 65535 + 1e-12


def test_render_constant_field_and_bad_kind(tmp_path):
    values, _ = load_render(render(np.ones((8, 8), complex), "magnitude", tmp_path / "c.png"))
    assert np.all(values == 1.0)
    with pytest.raises(ParameterError):
        render(np.ones((8, 8)), "intensity", tmp_path / "x.png")


def test_figures_written(tmp_path):
    assert plot_error_trace([1.0, 0.5, 0.1], tmp_path / "e.png").is_file()
    pos = np.random.default_rng(1).uniform(0, 50, (9, 2))
    assert plot_positions(pos, pos + 0.1, tmp_path / "p.png", truth=pos).is_file()
