"""CPU-side checks: the C-ABI library loads and exports every symbol the header
declares, host logic mirrors the reference, scene generators match the
reference goldens, and the dataset container round-trips."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native, errors, simulate
from paper_2205_04295_b200.engine import SolverConfig, _anchor, visit_order


def header_symbols():
    text = (ROOT / "include" / "ptycho_b200.h").read_text()
    return sorted(set(re.findall(r"PTY_API\s+\w+\s+(pty_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load(require_device=False)
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)
    assert lib.pty_abi_version() == 1


def test_workspace_sizes_are_consistent():
    lib = _native.load(require_device=False)
    a = lib.pty_sweep_workspace_bytes(0, 256, 3, 400, 1)
    b = lib.pty_sweep_workspace_bytes(1, 256, 3, 400, 1)
    assert 0 < a < b
    # scratch dominates: S * M * W^2 complex
    assert a >= 3 * 256 * 256 * 8
    assert lib.pty_sweep_workspace_bytes(0, 100, 3, 400, 1) == -1     # non power of two
    assert lib.pty_sweep_workspace_bytes(0, 256, 9, 400, 1) == -1     # > 8 modes
    assert lib.pty_register_scratch_bytes(256, 400, 10) > 0


def test_solver_config_validation_matches_reference():
    with pytest.raises(errors.ParameterError):
        SolverConfig(alpha_obj=1.5)
    with pytest.raises(errors.ParameterError):
        SolverConfig(beta=0.0)
    with pytest.raises(errors.ParameterError):
        SolverConfig(position_order="zigzag")
    with pytest.raises(errors.ParameterError):
        SolverConfig(mode_count=0)
    with pytest.raises(errors.ParameterError):
        SolverConfig(precision="fp16")
    with pytest.raises(ValueError):
        pk.PosRefConfig(beta1=1.0)
    with pytest.raises(ValueError):
        pk.PosRefConfig(sensor="XCORR_C")


def test_visit_order_and_anchors_match_goldens():
    for name in ("rpie", "epie_fixed", "posref_a"):
        g = golden(f"sweep_{name}")
        n = g["patterns"].shape[0]
        cfg = SolverConfig(position_order="fixed" if name == "epie_fixed" else "shuffled")
        for s in range(int(g["sweeps"])):
            np.testing.assert_array_equal(visit_order(n, cfg, s), g["orders"][s])
    # Python round(): half to even, as the reference's _anchor (engine.py:69-70)
    assert _anchor((10.5, 11.5)) == (12, 10)
    assert _anchor((-0.5, 2.5)) == (2, 0)


def test_status_word_maps_to_reference_exceptions():
    cases = [(errors.PTY_ERR_BOUNDS, errors.BoundsError),
             (errors.PTY_ERR_PROBE_ZERO, errors.DegenerateInputError),
             (errors.PTY_ERR_OBJECT_ZERO, errors.DegenerateInputError),
             (errors.PTY_ERR_NEGATIVE_I, errors.DataError),
             (errors.PTY_ERR_ARGUMENT, errors.ParameterError),
             (errors.PTY_ERR_CUDA, errors.NativeError)]
    for bit, exc in cases:
        with pytest.raises(exc):
            errors.raise_for_status(bit)
    errors.raise_for_status(0)
    assert issubclass(errors.BoundsError, IndexError)


def test_scene_generators_match_reference():
    g = golden("simulate")
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 32)
    plan = simulate.make_scan((4, 4), 7.0, 1.0, seed=3)
    np.testing.assert_array_equal(plan.nominal, g["nominal"])
    np.testing.assert_array_equal(plan.true_positions, g["true"])
    obj = simulate.make_object(simulate.canvas_shape_for(plan, 32), "spokes", seed=3)
    np.testing.assert_allclose(obj, g["obj"], rtol=0, atol=1e-14)
    probes = simulate.make_probe(simulate.ProbeSpec(2, (0.7, 0.3), "disk", 8.0), geom)
    np.testing.assert_allclose(np.stack(probes), g["probes"], rtol=0, atol=1e-14)
    plan1 = simulate.make_scan((10, 10), 16.0, 1.0, seed=1)
    np.testing.assert_array_equal(plan1.nominal, g["c1_positions"])


def test_dataset_round_trip(tmp_path):
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 16)
    rng = np.random.default_rng(0)
    ds = pk.PtychoDataset(patterns=rng.random((3, 16, 16)), positions=rng.random((3, 2)) * 4,
                          geometry=geom, seed=5)
    pk.write_dataset(tmp_path / "d", ds)
    back = pk.read_dataset(tmp_path / "d")
    np.testing.assert_array_equal(back.patterns, ds.patterns.astype(np.float32))
    np.testing.assert_array_equal(back.positions, ds.positions)
    assert back.geometry == geom and back.seed == 5
    (tmp_path / "d" / "patterns.raw").write_bytes(b"123")
    with pytest.raises(errors.DatasetIOError):
        pk.read_dataset(tmp_path / "d")


def test_reference_datasets_are_readable(tmp_path):
    """A dataset written by the reference's container format parses here."""
    g = golden("sweep_rpie")
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, int(g["window"]))
    ds = pk.PtychoDataset(patterns=g["patterns"], positions=g["positions_in"], geometry=geom)
    pk.write_dataset(tmp_path / "r", ds)
    back = pk.read_dataset(tmp_path / "r")
    np.testing.assert_array_equal(back.patterns, g["patterns"].astype(np.float64))


def test_integration_stub_structs_match_the_abi():
    """INTEGRATION.md's maintainer stub declares the same PtySlot / PtySweepArgs
    layout as the package's binding (field names, offsets, sizes)."""
    import ctypes as C
    import re
    from pathlib import Path
    from paper_2205_04295_b200 import _native
    text = (Path(__file__).resolve().parents[1] / "INTEGRATION.md").read_text()
    code = re.search(r"```python\n# ptychokit/_b200.py.*?\n(.*?)```", text, re.S).group(1)
    code = code.split("lib.pty_sweep.argtypes")[0].replace('lib = C.CDLL("libptycho_b200.so")', "")
    ns = {}
    exec(code, ns)
    for name in ("PtySlot", "PtySweepArgs"):
        a, b = ns[name], getattr(_native, name)
        assert C.sizeof(a) == C.sizeof(b), name
        assert [f[0] for f in a._fields_] == [f[0] for f in b._fields_], name
        for f in a._fields_:
            assert getattr(a, f[0]).offset == getattr(b, f[0]).offset, (name, f[0])
