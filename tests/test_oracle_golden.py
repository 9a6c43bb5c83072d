"""Pin the CPU oracle to the reference: every golden vector in tests/golden was
produced by running the reference (tests/golden/make_golden.py); the oracle
must reproduce them at fp64 round-off."""

import ast
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import golden
from oracle import batched, registration as oreg, rpie

SOLVER_DEFAULTS = dict(alpha_obj=0.9, alpha_probe=0.9, beta=1.0, gamma=1.0, mode_count=1,
                       iterations=100, position_order="shuffled", shuffle_seed=0,
                       init_seed=0, epsilon_rel=1e-12, ortho_interval=0,
                       update_probe_modes=True, posref=None, track_modulus_error=False)
POSREF_DEFAULTS = dict(sensor="XCORR_A", step_size=0.5, beta1=0.9, beta2=0.999,
                       eps_adam=1e-8, warmup_iterations=10, kappa=100, max_correction=1.0)


def cfg_from_repr(text):
    """Rebuild the generator's config dict (PosRefConfig(...) calls included)."""
    tree = ast.parse(text, mode="eval").body
    out = {}
    for k, v in zip(tree.keys, tree.values):
        if isinstance(v, ast.Call):
            kw = {a.arg: ast.literal_eval(a.value) for a in v.keywords}
            out[k.value] = SimpleNamespace(**{**POSREF_DEFAULTS, **kw})
        else:
            out[k.value] = ast.literal_eval(v)
    return SimpleNamespace(**{**SOLVER_DEFAULTS, **out})


def test_propagate_matches_reference():
    g = golden("fields")
    for w in (32, 64):
        np.testing.assert_allclose(rpie.centered_fft2(g[f"in_{w}"]), g[f"fwd_{w}"],
                                   rtol=0, atol=1e-14)
        np.testing.assert_allclose(rpie.centered_fft2(g[f"in_{w}"], inverse=True),
                                   g[f"bwd_{w}"], rtol=0, atol=1e-14)


def test_visit_matches_reference():
    g = golden("visit")
    probes = list(g["probes"])
    corrected, det, _ = rpie.modulus_project(probes, g["o"], g["I"])
    np.testing.assert_allclose(np.stack(corrected), g["corrected"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(np.stack(det), g["det"], rtol=1e-12, atol=1e-15)
    for k in range(4):
        beta, gamma = float(g[f"beta_{k}"]), float(g[f"gamma_{k}"])
        new_o = rpie.object_step(g["o"], probes, corrected, 0.9, gamma)
        new_p = [rpie.probe_step(p, g["o"], c, 0.8, beta) for p, c in zip(probes, corrected)]
        np.testing.assert_allclose(new_o, g[f"new_o_{k}"], rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(np.stack(new_p), g[f"new_p_{k}"], rtol=1e-12, atol=1e-15)


SWEEP_CASES = ["rpie", "epie_fixed", "ortho_mod", "noprobe", "posref_a", "posref_b"]


@pytest.mark.parametrize("name", SWEEP_CASES)
def test_sweep_trajectory_matches_reference(name):
    g = golden(f"sweep_{name}")
    cfg = cfg_from_repr(str(g["cfg_repr"]))
    w = int(g["window"])
    patterns = g["patterns"].astype(np.float64)
    st = rpie.initialize(patterns, g["positions_in"], w, cfg)
    assert tuple(st.canvas_origin) == tuple(g["canvas_origin"])
    np.testing.assert_array_equal(st.obj, g["init_obj"])
    np.testing.assert_allclose(np.stack(st.probes), g["init_probes"], rtol=0, atol=1e-13)
    for s in range(int(g["sweeps"])):
        order = rpie.visit_order(len(patterns), cfg.position_order, cfg.shuffle_seed,
                                 st.iteration)
        np.testing.assert_array_equal(order, g["orders"][s])
        rpie.sweep(st, patterns, w, cfg)
        scale = np.abs(g[f"s{s + 1}_obj"]).max()
        np.testing.assert_allclose(st.obj, g[f"s{s + 1}_obj"], rtol=0, atol=1e-11 * scale)
        pscale = np.abs(g[f"s{s + 1}_probes"]).max()
        np.testing.assert_allclose(np.stack(st.probes), g[f"s{s + 1}_probes"], rtol=0,
                                   atol=1e-11 * pscale)
        np.testing.assert_allclose(st.positions, g[f"s{s + 1}_positions"], rtol=0, atol=1e-12)
        if cfg.posref is not None:
            np.testing.assert_array_equal(st.adam_t, g[f"s{s + 1}_adam_t"])
            np.testing.assert_allclose(st.adam_m, g[f"s{s + 1}_adam_m"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(st.error_trace, g["error_trace"], rtol=1e-10)
    if cfg.track_modulus_error:
        assert max(st.modulus_error_trace) <= 1e-9
        assert max(g["modulus_error_trace"]) <= 1e-9


def test_batched_b1_is_the_reference_sweep():
    """The (unpinned) batched extension collapses to the reference at b=1."""
    for name in ("rpie", "posref_a"):
        g = golden(f"sweep_{name}")
        cfg = cfg_from_repr(str(g["cfg_repr"]))
        w = int(g["window"])
        patterns = g["patterns"].astype(np.float64)
        a = rpie.initialize(patterns, g["positions_in"], w, cfg)
        b = a.copy()
        for _ in range(int(g["sweeps"])):
            rpie.sweep(a, patterns, w, cfg)
            batched.sweep_batched(b, patterns, w, cfg, batch=1)
        np.testing.assert_array_equal(a.obj, b.obj)
        np.testing.assert_array_equal(np.stack(a.probes), np.stack(b.probes))
        np.testing.assert_array_equal(a.positions, b.positions)
        assert a.error_trace == b.error_trace


def test_registration_matches_reference():
    g = golden("registration")
    for pair, weighting, kappa, dy, dx, peak in g["rows"]:
        k = int(pair)
        est = oreg.register(g[f"ref_{k}"], g[f"mov_{k}"], ["phase", "raw"][int(weighting)],
                            int(kappa))
        assert (est.dy, est.dx) == (dy, dx)
        assert est.peak_value == pytest.approx(peak, rel=1e-10)
    est = oreg.coarse_shift(g["tie_xps"])
    assert (est.dy, est.dx) == tuple(g["tie_est"][:2])


def test_adam_matches_reference():
    g = golden("adam")
    pc = SimpleNamespace(**{**POSREF_DEFAULTS, "step_size": 0.3, "beta1": 0.8,
                            "beta2": 0.95, "max_correction": 10})
    m, v, t = np.zeros((3, 2)), np.zeros((3, 2)), np.zeros(3, np.int64)
    for step in range(g["g"].shape[0]):
        for j in range(3):
            d = rpie.adam_update(m, v, t, j, tuple(g["g"][step, j]), pc)
            np.testing.assert_array_equal(d, g["delta"][step, j])
    np.testing.assert_array_equal(m, g["m"])
    np.testing.assert_array_equal(t, g["t"])
    pos = g["pos_in"].copy()
    for j, dlt in enumerate([(0.25, -0.5), (0.5, -0.5), (-3.0, 4.0)]):
        rpie.clamp_move(pos, j, dlt, (0.0, 0.0, 10.0, 10.0))
    np.testing.assert_array_equal(pos, g["pos_out"])
