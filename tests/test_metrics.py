"""Quality metrics (metrics.py:20-75) against goldens produced by the reference
itself (tests/golden/make_golden.py gen_metrics).  The functions are
device-agnostic torch code: the CPU tests run them on host tensors, the GPU
test on the reconstruction's device."""

import numpy as np
import pytest

from conftest import golden
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import metrics


def _check(device):
    import torch
    g = golden("metrics")
    probes = torch.as_tensor(g["probes"], device=device)
    recon = torch.as_tensor(g["recon"], device=device)
    for thr in (0.05, 0.3):
        mask = metrics.coverage_mask(probes, g["positions"], g["recon"].shape, g["canvas_origin"], thr)
        assert np.array_equal(mask.cpu().numpy(), g[f"mask_{thr}"])
        e = metrics.object_error(recon, g["truth"], mask)
        assert e == pytest.approx(float(g[f"object_error_{thr}"][0]), rel=1e-12, abs=1e-15)
    assert metrics.position_rmse(g["est"], g["true"]) == pytest.approx(float(g["position_rmse"][0]), rel=1e-13)


def test_metrics_match_reference_cpu():
    _check("cpu")


def test_metrics_errors():
    with pytest.raises(pk.errors.ShapeError):
        metrics.object_error(np.ones((3, 3)), np.ones((3, 4)), np.ones((3, 3), bool))
    with pytest.raises(pk.errors.DegenerateInputError):
        metrics.object_error(np.ones((3, 3)), np.ones((3, 3)), np.zeros((3, 3), bool))
    with pytest.raises(pk.errors.DegenerateInputError):
        metrics.object_error(np.zeros((3, 3)), np.ones((3, 3)), np.ones((3, 3), bool))
    with pytest.raises(pk.errors.ShapeError):
        metrics.position_rmse(np.zeros((3, 2)), np.zeros((4, 2)))


def test_metrics_report_json(tmp_path):
    r = metrics.MetricsReport(error_trace=[0.5, 0.25], position_rmse=0.1)
    import json
    assert json.loads(r.to_json(tmp_path / "m.json").read_text())["error_trace"] == [0.5, 0.25]


@pytest.mark.gpu
def test_metrics_match_reference_gpu(gpu):
    _check("cuda")
