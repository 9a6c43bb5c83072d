"""Opt-in subpixel reconstruction gather (SolverConfig.subpixel_gather; the
extension of SURVEY.md 8(a) row a4): the crop of every visit is the
simulator's extract_view (/root/reference/pkg/src/ptychokit/simulate.py:157-166,
fields.py:110-122) at the float position and the object update is shifted back
before the paste.  Parity is unpinned against the reference (no such mode);
it is pinned to its CPU statement oracle/rpie.py sweep(subpixel_gather) in
fp64, and to the reference path itself when every residual is zero."""

import numpy as np
import pytest

import paper_2205_04295_b200 as pk
from oracle import rpie
from test_gpu_parity import rel_l2

pytestmark = pytest.mark.gpu


def scene(w=32, m=2, grid=(4, 4), jitter=1.0, seed=7):
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, w)
    plan = pk.make_scan(grid, w / 5, jitter, seed=seed)
    obj = pk.make_object(pk.canvas_shape_for(plan, w), "spokes", seed=seed)
    powers = (1.0,) if m == 1 else (0.8, 0.2)
    probes = pk.make_probe(pk.ProbeSpec(m, powers, "disk", w * 0.25), geom)
    ds = pk.synthesize(obj, probes, plan, geom)
    ds.patterns = ds.patterns.astype(np.float32).astype(np.float64)
    # reconstruct at the TRUE (subpixel) positions: the gather must interpolate
    ds.positions = plan.true_positions.copy()
    return ds


@pytest.mark.parametrize("posref", [None, "XCORR_A", "XCORR_B"])
def test_subpixel_gather_fp64_matches_oracle(gpu, posref):
    ds = scene()
    assert np.any(ds.positions != np.round(ds.positions))
    pc = None if posref is None else pk.PosRefConfig(sensor=posref, kappa=10, warmup_iterations=1)
    cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=2,
                          precision="fp64", subpixel_gather=True, posref=pc)
    st = pk.initialize(ds, cfg)
    ost = rpie.initialize(ds.patterns, ds.positions, 32, cfg)
    for _ in range(3):
        pk.sweep(st, ds, cfg)
        rpie.sweep(ost, ds.patterns, 32, cfg)
    e_o = rel_l2(st.obj.cpu().numpy(), ost.obj)
    e_p = rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes))
    print(f"PARITY subpixel fp64 posref={posref}: obj {e_o:.3e} probe {e_p:.3e}")
    assert e_o < 1e-9 and e_p < 1e-9
    np.testing.assert_allclose(st.positions.cpu().numpy(), ost.positions, rtol=0, atol=1e-9)
    np.testing.assert_allclose(st.error_trace, ost.error_trace, rtol=1e-9)


def test_subpixel_gather_fp32_and_quality(gpu):
    """fp32 within the north-star tolerance of the fp64 oracle, and the
    subpixel gather fits subpixel-jittered data better than integer crops."""
    ds = scene(w=64, grid=(5, 5), seed=3)
    base = dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=2)
    cfg = pk.SolverConfig(**base, precision="fp32", subpixel_gather=True)
    st = pk.initialize(ds, cfg)
    ost = rpie.initialize(ds.patterns, ds.positions, 64, cfg)
    for _ in range(2):
        pk.sweep(st, ds, cfg)
        rpie.sweep(ost, ds.patterns, 64, cfg)
    assert rel_l2(st.obj.cpu().numpy(), ost.obj) < 1e-4
    assert rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)) < 1e-4
    plain = pk.initialize(ds, pk.SolverConfig(**base, precision="fp32"))
    for _ in range(8):
        pk.sweep(st, ds, cfg)
        pk.sweep(plain, ds, pk.SolverConfig(**base, precision="fp32"))
    assert st.error_trace[-1] < plain.error_trace[-1]


def test_subpixel_on_integer_grid_is_the_reference_path(gpu):
    """Every residual zero: the subpixel mode reduces to the reference sweep
    (oracle without the extension) to fp64 round-off."""
    ds = scene(jitter=0.0)
    ds.positions = np.round(ds.positions)
    cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=2,
                          precision="fp64", subpixel_gather=True)
    ref = pk.SolverConfig(**{**cfg.__dict__, "subpixel_gather": False})
    st = pk.initialize(ds, cfg)
    ost = rpie.initialize(ds.patterns, ds.positions, 32, ref)
    for _ in range(2):
        pk.sweep(st, ds, cfg)
        rpie.sweep(ost, ds.patterns, 32, ref)
    assert rel_l2(st.obj.cpu().numpy(), ost.obj) < 1e-12
    assert rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)) < 1e-12


def test_default_off_is_bit_identical(gpu):
    """subpixel_gather defaults to False and leaves the fused sweep untouched."""
    ds = scene()
    a = pk.SolverConfig(mode_count=2, alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5)
    b = pk.SolverConfig(**{**a.__dict__, "subpixel_gather": False})
    assert a.subpixel_gather is False
    s1, s2 = pk.initialize(ds, a), pk.initialize(ds, b)
    for _ in range(2):
        pk.sweep(s1, ds, a)
        pk.sweep(s2, ds, b)
    assert np.array_equal(s1.obj.cpu().numpy(), s2.obj.cpu().numpy())
    assert np.array_equal(s1.probe_stack.cpu().numpy(), s2.probe_stack.cpu().numpy())
    assert s1.error_trace == s2.error_trace


def test_subpixel_config_validation(gpu):
    with pytest.raises(pk.errors.ParameterError):
        pk.SolverConfig(subpixel_gather=True, batch_size=4)
    with pytest.raises(pk.errors.ParameterError):
        pk.SolverConfig(subpixel_gather=True, track_modulus_error=True)
