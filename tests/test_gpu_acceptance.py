"""Quality tier Q: the reference's own acceptance criteria 3 and 6
(/root/reference/pkg/tests/test_acceptance.py:142-163, 249-292), run through
the CUDA path (default fp32) with the same scenes, seeds, thresholds and
metrics (paper_2205_04295_b200.metrics == ptychokit.metrics, tests/test_metrics.py)."""

import numpy as np
import pytest

import paper_2205_04295_b200 as pk
from paper_2205_04295_b200.metrics import coverage_mask, object_error, position_rmse

pytestmark = pytest.mark.gpu

GEOM64 = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 64)


def recon_object_error(state, dataset) -> float:
    """test_acceptance.py:28-41."""
    mask = coverage_mask(state.probes, state.positions, tuple(state.obj.shape), state.canvas_origin)
    truth = dataset.ground_truth.obj
    r0, c0 = state.canvas_origin
    h, w = state.obj.shape
    ra, ca = max(r0, 0), max(c0, 0)
    rb, cb = min(r0 + h, truth.shape[0]), min(c0 + w, truth.shape[1])
    return object_error(state.obj[ra - r0:rb - r0, ca - c0:cb - c0],
                        truth[ra:rb, ca:cb], mask[ra - r0:rb - r0, ca - c0:cb - c0])


def test_criterion_3_noiseless_recovery(gpu):
    plan = pk.make_scan((9, 9), 9.0, 0.5, seed=5)
    obj = pk.make_object(pk.canvas_shape_for(plan, 64), "spokes", seed=5)
    probes = pk.make_probe(pk.ProbeSpec(1, (1.0,), "disk", 15.0), GEOM64)
    ds = pk.synthesize(obj, probes, plan, GEOM64, noise="none", seed=5)
    ds.positions[:] = ds.ground_truth.true_positions
    cfg = pk.SolverConfig(iterations=200, update_probe_modes=False)
    state = pk.initialize(ds, cfg)
    state.probes = [p.copy() for p in probes]
    err = np.inf
    for _ in range(200):
        pk.sweep(state, ds, cfg)
        err = min(err, recon_object_error(state, ds))
        if err < 1e-3:
            break
    assert err < 1e-3, f"object error {err:.2e} after {state.iteration} iterations"


def test_criterion_6_position_refinement(gpu):
    plan = pk.make_scan((7, 7), 10.0, 3.0, seed=7)
    plan.true_positions[:] = np.round(plan.true_positions)
    obj = pk.make_object(pk.canvas_shape_for(plan, 64), "spokes", seed=7)
    probes = pk.make_probe(pk.ProbeSpec(1, (1.0,), "disk", 20.0), GEOM64)
    ds = pk.synthesize(obj, probes, plan, GEOM64, noise="none", seed=7)
    true = ds.ground_truth.true_positions
    corrupt = true + np.random.default_rng(42).uniform(-2, 2, true.shape)
    initial_rmse = position_rmse(corrupt, true)

    def run(sensor, step_size):
        posref = None
        if sensor is not None:
            posref = pk.PosRefConfig(sensor=sensor, step_size=step_size, warmup_iterations=10, kappa=100)
        ds.positions[:] = corrupt
        cfg = pk.SolverConfig(iterations=150, shuffle_seed=3, posref=posref, update_probe_modes=False)
        state = pk.initialize(ds, cfg)
        state.probes = [p.copy() for p in probes]
        for _ in range(150):
            pk.sweep(state, ds, cfg)
        return position_rmse(state.positions, true), recon_object_error(state, ds)

    rmse_a, objerr_a = run("XCORR_A", 0.2)
    _, objerr_off = run(None, 0.0)
    rmse_b, _ = run("XCORR_B", 0.2)
    assert rmse_a <= 0.30 * initial_rmse, (rmse_a, initial_rmse)
    assert objerr_a <= 0.5 * objerr_off, (objerr_a, objerr_off)
    assert rmse_b > rmse_a
