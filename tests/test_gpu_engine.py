"""The reference's engine / simulate behaviour tests
(/root/reference/pkg/tests/test_engine.py:64-224, test_simulate.py:136-185)
restated against the CUDA path: initialisation, clean-scene convergence,
Poisson robustness, ordering, run/checkpoint, and the GPU virtual experiment
pinned to the reference's own patterns (tests/golden/simulate.npz)."""

import numpy as np
import pytest

from conftest import golden
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import dataio, errors

pytestmark = pytest.mark.gpu

GEOM = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 32)


def scene(mode_count=1, powers=(1.0,), noise="none", grid=(4, 4), step=7.0, jitter=0.0, seed=3, **synth):
    """test_engine.py:18-24."""
    plan = pk.make_scan(grid, step, jitter, seed=seed)
    obj = pk.make_object(pk.canvas_shape_for(plan, 32), "spokes", seed=seed)
    probes = pk.make_probe(pk.ProbeSpec(mode_count, powers, "disk", 8.0), GEOM)
    ds = pk.synthesize(obj, probes, plan, GEOM, noise=noise, seed=seed, **synth)
    return obj, probes, plan, ds


def ifft_c(a):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(a), norm="ortho"))


def host(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


# ------------------------------------------------------------- simulate ----
def test_synthesize_matches_reference_patterns(gpu):
    """simulate.py:157-198 on the GPU (fp64) vs the reference's own output for
    the same seeded scene (subpixel-shifted views, 2 modes)."""
    g = golden("simulate")
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 32)
    plan = pk.make_scan((4, 4), 7.0, 1.0, seed=3)
    np.testing.assert_array_equal(plan.true_positions, g["true"])
    obj = pk.make_object(pk.canvas_shape_for(plan, 32), "spokes", seed=3)
    probes = pk.make_probe(pk.ProbeSpec(2, (0.7, 0.3), "disk", 8.0), geom)
    ds = pk.synthesize(obj, probes, plan, geom)
    ref = g["patterns"]
    assert np.abs(ds.patterns - ref).max() <= 1e-12 * np.abs(ref).max()


def test_synthesize_parseval_and_uniform_object(gpu):
    """test_simulate.py:140-155: unitary propagation; a uniform object gives
    position-independent patterns equal to |propagate(P)|^2."""
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 64)
    plan = pk.make_scan((2, 2), 10.0, 0.0, seed=0)
    obj = np.ones(pk.canvas_shape_for(plan, 64), dtype=complex)
    probes = pk.make_probe(pk.ProbeSpec(1, (1.0,), "disk", 12.0), geom)
    ds = pk.synthesize(obj, probes, plan, geom)
    want = np.abs(host(pk.propagate(probes[0]))) ** 2
    for j in range(4):
        np.testing.assert_allclose(ds.patterns[j], want, atol=1e-12)
        assert ds.patterns[j].sum() == pytest.approx(np.sum(np.abs(probes[0]) ** 2), rel=1e-12)


def test_poisson_noise_totals_and_determinism(gpu):
    """test_simulate.py:164-178."""
    _, _, _, clean = scene(noise="none", seed=4)
    _, _, _, a = scene(noise="poisson", seed=4, photon_budget=1e6)
    _, _, _, b = scene(noise="poisson", seed=4, photon_budget=1e6)
    for j in range(a.n_positions):
        assert a.patterns[j].sum() == pytest.approx(clean.patterns[j].sum(), rel=5e-3)
    assert np.any(a.patterns != clean.patterns) and np.all(a.patterns >= 0)
    np.testing.assert_array_equal(a.patterns, b.patterns)
    with pytest.raises(errors.ParameterError):
        scene(noise="gaussian")


# ----------------------------------------------------------- initialize ----
def test_initialize_object_canvas_and_probes(gpu):
    """test_engine.py:65-95: unit object on the anchor bounding box, first probe
    = back-propagated mean amplitude, extra modes orthogonal at 1 % power,
    positions a private copy."""
    _, _, _, ds = scene()
    st = pk.initialize(ds, pk.SolverConfig(precision="fp64"))
    assert np.all(host(st.obj) == 1.0)
    anchors = np.stack([(round(p[1]), round(p[0])) for p in ds.positions])
    assert tuple(st.obj.shape) == tuple(anchors.max(axis=0) - anchors.min(axis=0) + 32)
    assert st.canvas_origin == tuple(int(v) for v in anchors.min(axis=0))
    want = ifft_c(np.sqrt(ds.patterns.mean(axis=0)).astype(complex))
    np.testing.assert_allclose(host(st.probes[0]), want, atol=1e-12)
    st3 = pk.initialize(ds, pk.SolverConfig(mode_count=3, precision="fp64"))
    pr = [host(p) for p in st3.probes]
    p1 = np.sum(np.abs(pr[0]) ** 2)
    for k in (1, 2):
        assert np.sum(np.abs(pr[k]) ** 2) == pytest.approx(0.01 * p1, rel=1e-10)
        for prev in pr[:k]:
            assert abs(np.vdot(prev, pr[k])) < 1e-10 * p1
    st.positions[0, 0] += 1.0
    assert ds.positions[0, 0] != float(st.positions[0, 0])


# ---------------------------------------------------------------- sweep ----
def test_error_trace_decreases_on_clean_scene(gpu):
    """test_engine.py:144-153."""
    _, _, _, ds = scene()
    cfg = pk.SolverConfig(iterations=30)
    st = pk.initialize(ds, cfg)
    for _ in range(30):
        pk.sweep(st, ds, cfg)
    assert st.error_trace[-1] < 0.4 * st.error_trace[0]
    trace = np.asarray(st.error_trace)
    assert trace[10:].max() < trace[:10].max()


def test_no_nan_on_poisson_data(gpu):
    """test_engine.py:196-205."""
    _, _, _, ds = scene(noise="poisson", photon_budget=1e5)
    cfg = pk.SolverConfig(mode_count=2)
    st = pk.initialize(ds, cfg)
    for _ in range(25):
        pk.sweep(st, ds, cfg)
    assert np.all(np.isfinite(host(st.obj)))
    assert all(np.all(np.isfinite(host(p))) for p in st.probes)
    assert np.all(np.isfinite(st.error_trace))


def test_shuffle_order_depends_on_seed(gpu):
    """test_engine.py:180-186."""
    _, _, _, ds = scene()
    a = pk.initialize(ds, pk.SolverConfig(shuffle_seed=0))
    b = pk.initialize(ds, pk.SolverConfig(shuffle_seed=1))
    pk.sweep(a, ds, pk.SolverConfig(shuffle_seed=0))
    pk.sweep(b, ds, pk.SolverConfig(shuffle_seed=1))
    assert np.any(host(a.obj) != host(b.obj))


def test_deterministic_rerun_with_posref_on_poisson_data(gpu):
    """test_engine.py:164-178."""
    _, _, _, ds = scene(noise="poisson")
    cfg = pk.SolverConfig(iterations=5, mode_count=2, posref=pk.PosRefConfig(warmup_iterations=2))
    runs = []
    for _ in range(2):
        st = pk.initialize(ds, cfg)
        for _ in range(5):
            pk.sweep(st, ds, cfg)
        runs.append(st)
    np.testing.assert_array_equal(host(runs[0].obj), host(runs[1].obj))
    np.testing.assert_array_equal(host(runs[0].positions), host(runs[1].positions))
    for a, b in zip(runs[0].probes, runs[1].probes):
        np.testing.assert_array_equal(host(a), host(b))
    assert runs[0].error_trace == runs[1].error_trace


def test_run_and_checkpointing(gpu, tmp_path):
    """test_engine.py:208-224, plus the Adam buffers this package checkpoints."""
    _, _, _, ds = scene()
    st = pk.run(ds, pk.SolverConfig(iterations=4))
    assert st.iteration == 4 and len(st.seconds_per_iteration) == 4
    cfg = pk.SolverConfig(iterations=4, posref=pk.PosRefConfig(warmup_iterations=1))
    st = pk.run(ds, cfg, checkpoint_every=2, checkpoint_dir=tmp_path)
    back = dataio.read_checkpoint(tmp_path / "iter_0002")
    assert back["iteration"] == 2 and len(back["error_trace"]) == 2
    last = dataio.read_checkpoint(tmp_path / "iter_0004")
    np.testing.assert_array_equal(last["positions"], host(st.positions))
    np.testing.assert_array_equal(last["adam"][2], host(st.adam.t))


def test_resume_from_checkpoint_continues_the_run(gpu, tmp_path):
    """run 4 sweeps with checkpoints, resume from iteration 2 and sweep twice:
    same visit orders, positions and Adam counters as the uninterrupted run;
    fields within complex64 container rounding."""
    _, _, _, ds = scene(jitter=1.0)
    cfg = pk.SolverConfig(iterations=4, posref=pk.PosRefConfig(warmup_iterations=1, kappa=10))
    full = pk.run(ds, cfg, checkpoint_every=2, checkpoint_dir=tmp_path)
    st = pk.resume(tmp_path / "iter_0002", ds, cfg)
    assert st.iteration == 2
    for _ in range(2):
        pk.sweep(st, ds, cfg)
    np.testing.assert_array_equal(host(st.adam.t), host(full.adam.t))
    np.testing.assert_allclose(host(st.positions), host(full.positions), atol=1e-6)
    np.testing.assert_allclose(host(st.obj), host(full.obj), atol=1e-5)
    np.testing.assert_allclose(st.error_trace, full.error_trace, rtol=1e-4)
