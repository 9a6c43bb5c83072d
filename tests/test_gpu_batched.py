"""Batched (semi-parallel) extension on the GPU (pty_batch_contrib/apply).

Parity is unpinned against the reference (no batched mode there); it is pinned
(1) to the reference itself at batch size 1 -- the batched kernels must equal
the sequential sweep kernel bit for bit -- and (2) to the CPU statement of the
extension (oracle/batched.py) at b > 1 in fp64."""

import numpy as np
import pytest

from conftest import golden
import paper_2205_04295_b200 as pk
from oracle import batched, rpie
from test_gpu_parity import make_ds, pkg_cfg, rel_l2
from test_oracle_golden import cfg_from_repr

pytestmark = pytest.mark.gpu


def _cfg(name, precision, batch):
    g = golden(f"sweep_{name}")
    c = pkg_cfg(cfg_from_repr(str(g["cfg_repr"])), precision)
    return g, pk.SolverConfig(**{**c.__dict__, "batch_size": batch})


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-13), ("fp32", 2e-6)])
def test_batch_of_one_is_the_sequential_kernel(gpu, precision, tol):
    """b = 1 through pty_batch_* == the reference-order sweep kernel up to
    round-off (the two kernels evaluate the same expressions but the compiler
    contracts FMAs differently; bit-exact b=1 equivalence with the reference is
    proven on the CPU statement, test_oracle_golden.py)."""
    for name in ("rpie", "ortho_mod"):
        g, seq = _cfg(name, precision, 1)
        bat = pk.SolverConfig(**{**seq.__dict__, "batch_size": 1})
        ds = make_ds(g["patterns"], g["positions_in"], g["window"])
        a = pk.initialize(ds, seq)
        b = pk.initialize(ds, seq)
        for _ in range(2):
            pk.sweep(a, ds, seq)
            pk.engine.sweep_batched(b, ds, bat)
        assert rel_l2(b.obj.cpu().numpy(), a.obj.cpu().numpy()) < tol, name
        assert rel_l2(b.probe_stack.cpu().numpy(), a.probe_stack.cpu().numpy()) < 10 * tol, name
        np.testing.assert_allclose(a.error_trace, b.error_trace, rtol=10 * tol)


@pytest.mark.parametrize("name,batch", [("rpie", 4), ("rpie", 16), ("epie_fixed", 5),
                                        ("noprobe", 3), ("posref_a", 6), ("posref_b", 4)])
def test_fp64_batched_matches_oracle(gpu, name, batch):
    g, cfg = _cfg(name, "fp64", batch)
    w = int(g["window"])
    ds = make_ds(g["patterns"], g["positions_in"], w)
    st = pk.initialize(ds, cfg)
    ost = rpie.initialize(ds.patterns, ds.positions, w, cfg)
    for _ in range(int(g["sweeps"])):
        pk.sweep(st, ds, cfg)
        batched.sweep_batched(ost, ds.patterns, w, cfg, batch)
    assert rel_l2(st.obj.cpu().numpy(), ost.obj) < 1e-9
    assert rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)) < 1e-9
    np.testing.assert_allclose(st.positions.cpu().numpy(), ost.positions, rtol=0, atol=1e-9)
    np.testing.assert_allclose(st.error_trace, ost.error_trace, rtol=1e-9)


def test_fp32_batched_matches_oracle(gpu):
    g, cfg = _cfg("rpie", "fp32", 8)
    w = int(g["window"])
    ds = make_ds(g["patterns"], g["positions_in"], w)
    st = pk.initialize(ds, cfg)
    ost = rpie.initialize(ds.patterns, ds.positions, w, cfg)
    pk.sweep(st, ds, cfg)
    batched.sweep_batched(ost, ds.patterns, w, cfg, 8)
    assert rel_l2(st.obj.cpu().numpy(), ost.obj) < 1e-5
    assert rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)) < 1e-4


def test_batched_rerun_is_bit_identical(gpu):
    g, cfg = _cfg("rpie", "fp32", 8)
    ds = make_ds(g["patterns"], g["positions_in"], g["window"])
    runs = []
    for _ in range(2):
        st = pk.initialize(ds, cfg)
        for _ in range(3):
            pk.sweep(st, ds, cfg)
        runs.append((st.obj.cpu().numpy(), st.probe_stack.cpu().numpy(), list(st.error_trace)))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]


def test_batched_errors(gpu):
    g, cfg = _cfg("rpie", "fp32", 4)
    ds = make_ds(g["patterns"], g["positions_in"], g["window"])
    st = pk.initialize(ds, cfg)
    st.probe_stack.zero_()
    with pytest.raises(pk.errors.DegenerateInputError):
        pk.sweep(st, ds, cfg)
    st = pk.initialize(ds, cfg)
    st.positions[3, 1] = -50.0
    with pytest.raises(pk.errors.BoundsError):
        pk.sweep(st, ds, cfg)
