"""Generate the golden vectors that pin the oracle (and the CUDA path) to the
reference.  Run HERE, where the read-only reference tree exists:

    python tests/golden/make_golden.py

It imports ``ptychokit`` from /root/reference/pkg/src (never copied), runs the
reference's own functions on seeded inputs and freezes inputs + outputs as
.npz fixtures in this directory.  The fixtures travel with the repo; the GPU
box never needs /root/reference.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def _ref():
    sys.path.insert(0, str(REF))
    import ptychokit.engine as engine
    import ptychokit.fields as fields
    import ptychokit.posref as posref
    import ptychokit.registration as registration
    import ptychokit.simulate as simulate
    import ptychokit.dataio as dataio
    return engine, fields, posref, registration, simulate, dataio


engine, fields, posref, registration, simulate, dataio = _ref()


def rt32(ds, tmp):
    """Round-trip a dataset through the reference container so patterns are
    float32-exact (dataio.py:92-93,159), as the GPU stores them."""
    dataio.write_dataset(tmp, ds)
    return dataio.read_dataset(tmp)


def scene(window, grid, step, radius, modes, powers, jitter, seed, kind="spokes",
          noise="none", photon_budget=1e6):
    g = fields.Geometry.create(8.3187e-10, 0.75, 20e-6, window)
    plan = simulate.make_scan(grid, step, jitter, seed=seed)
    obj = simulate.make_object(simulate.canvas_shape_for(plan, window), kind, seed=seed)
    probes = simulate.make_probe(simulate.ProbeSpec(modes, powers, "disk", radius), g)
    ds = simulate.synthesize(obj, probes, plan, g, noise=noise, seed=seed,
                             photon_budget=photon_budget)
    return g, plan, obj, probes, ds


def pattern_digest(patterns) -> str:
    return hashlib.sha256(np.ascontiguousarray(patterns, np.float32).tobytes()).hexdigest()


def smooth(side, seed, sigma=2.0):
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    return gaussian_filter(rng.standard_normal((side, side)), sigma)


def gen_fields():
    out = {}
    for w in (32, 64):
        rng = np.random.default_rng([7, w])
        f = rng.standard_normal((w, w)) + 1j * rng.standard_normal((w, w))
        out[f"in_{w}"] = f
        out[f"fwd_{w}"] = fields.propagate(f, "forward")
        out[f"bwd_{w}"] = fields.propagate(f, "backward")
    np.savez_compressed(OUT / "fields.npz", **out)


def gen_visit(tmp):
    _, _, obj, probes, ds = scene(64, (3, 3), 9.0, 16.0, 2, (0.7, 0.3), 0.0, 3)
    ds = rt32(ds, tmp / "visit")
    o_j = fields.crop(obj, fields.CropBox(2, 3, 64))
    i_j = ds.patterns[4]
    out = {"o": o_j, "probes": np.stack(probes), "I": i_j}
    for k, (beta, gamma) in enumerate([(1.0, 1.0), (0.5, 0.5), (0.3, 0.25), (0.9, 0.05)]):
        corrected, det = engine.magnitude_correct(probes, o_j, i_j)
        new_o = engine.update_object(o_j, probes, corrected, 0.9, gamma)
        new_p = [engine.update_probe(p, o_j, c, 0.8, beta) for p, c in zip(probes, corrected)]
        out[f"beta_{k}"] = beta
        out[f"gamma_{k}"] = gamma
        out[f"new_o_{k}"] = new_o
        out[f"new_p_{k}"] = np.stack(new_p)
    out["corrected"] = np.stack(corrected)
    out["det"] = np.stack(det)
    np.savez_compressed(OUT / "visit.npz", **out)


def _state_arrays(st, prefix, out):
    out[prefix + "obj"] = st.obj.copy()
    out[prefix + "probes"] = np.stack(st.probes)
    out[prefix + "positions"] = st.positions.copy()
    if st.adam is not None:
        out[prefix + "adam_m"] = st.adam.m.copy()
        out[prefix + "adam_v"] = st.adam.v.copy()
        out[prefix + "adam_t"] = st.adam.t.copy()


def gen_sweeps(tmp):
    """Short trajectories on small scenes, several solver configurations."""
    cases = {
        "rpie": dict(scene=dict(window=32, grid=(4, 4), step=7.0, radius=8.0, modes=2,
                                powers=(0.7, 0.3), jitter=1.0, seed=3),
                     cfg=dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5,
                              mode_count=2), sweeps=3),
        "epie_fixed": dict(scene=dict(window=32, grid=(4, 4), step=7.0, radius=8.0, modes=1,
                                      powers=(1.0,), jitter=1.0, seed=4),
                           cfg=dict(alpha_obj=0.9, alpha_probe=0.8, beta=1.0, gamma=1.0,
                                    position_order="fixed"), sweeps=3),
        "ortho_mod": dict(scene=dict(window=32, grid=(4, 4), step=7.0, radius=8.0, modes=3,
                                     powers=(0.6, 0.25, 0.15), jitter=1.0, seed=5),
                          cfg=dict(alpha_obj=0.8, alpha_probe=0.7, beta=0.3, gamma=0.25,
                                   mode_count=3, ortho_interval=2, track_modulus_error=True,
                                   shuffle_seed=4, init_seed=2), sweeps=4),
        "noprobe": dict(scene=dict(window=64, grid=(3, 3), step=12.0, radius=16.0, modes=1,
                                   powers=(1.0,), jitter=1.0, seed=6),
                        cfg=dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.9, gamma=0.05,
                                 update_probe_modes=False), sweeps=2),
        "posref_a": dict(scene=dict(window=32, grid=(5, 5), step=7.0, radius=8.0, modes=2,
                                    powers=(0.8, 0.2), jitter=1.0, seed=7),
                         cfg=dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5,
                                  mode_count=2,
                                  posref=posref.PosRefConfig(sensor="XCORR_A", kappa=10,
                                                             warmup_iterations=1)),
                         sweeps=4, perturb=2.0),
        "posref_b": dict(scene=dict(window=32, grid=(4, 4), step=7.0, radius=8.0, modes=1,
                                    powers=(1.0,), jitter=1.0, seed=8),
                         cfg=dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5,
                                  posref=posref.PosRefConfig(sensor="XCORR_B", kappa=20,
                                                             warmup_iterations=1)),
                         sweeps=3, perturb=1.5),
    }
    for name, case in cases.items():
        _, plan, _, _, ds = scene(**case["scene"])
        ds = rt32(ds, tmp / name)
        if "perturb" in case:
            rng = np.random.default_rng(42)
            ds.positions = ds.positions + rng.uniform(-case["perturb"], case["perturb"],
                                                      ds.positions.shape)
            # keep every nominal crop inside the initial canvas bounding box
        cfg = engine.SolverConfig(**case["cfg"])
        st = engine.initialize(ds, cfg)
        out = {"patterns": ds.patterns.astype(np.float32), "positions_in": ds.positions,
               "window": ds.geometry.window, "sweeps": case["sweeps"]}
        _state_arrays(st, "init_", out)
        out["canvas_origin"] = np.array(st.canvas_origin)
        orders = []
        for s in range(case["sweeps"]):
            if cfg.position_order == "shuffled":
                orders.append(np.random.default_rng([cfg.shuffle_seed, st.iteration])
                              .permutation(ds.n_positions))
            else:
                orders.append(np.arange(ds.n_positions))
            engine.sweep(st, ds, cfg)
            _state_arrays(st, f"s{s + 1}_", out)
        out["orders"] = np.stack(orders)
        out["error_trace"] = np.array(st.error_trace)
        out["modulus_error_trace"] = np.array(st.modulus_error_trace)
        out["cfg_repr"] = repr(case["cfg"])
        np.savez_compressed(OUT / f"sweep_{name}.npz", **out)


def gen_registration():
    out = {}
    rows = []   # (pair, weighting 0=phase 1=raw, kappa, dy, dx, peak)
    k = 0
    for side in (16, 32, 64):
        for seed in range(3):
            ref = smooth(side, 100 + seed + side)
            rng = np.random.default_rng(200 + seed + side)
            dx, dy = rng.uniform(-3, 3, 2)
            out[f"ref_{k}"] = ref
            out[f"mov_{k}"] = fields.subpixel_shift(ref, dx, dy).real
            for weighting in ("phase", "raw"):
                for kappa in (1, 10, 20, 100):
                    est = registration.register(out[f"ref_{k}"], out[f"mov_{k}"],
                                                weighting, kappa)
                    rows.append((k, 0 if weighting == "phase" else 1, kappa,
                                 est.dy, est.dx, est.peak_value))
            k += 1
    # complex (XCORR_A-like) pairs
    for seed in range(3):
        o = simulate.make_object((32, 32), "phase-screen", seed=seed + 3)
        out[f"ref_{k}"] = o
        out[f"mov_{k}"] = fields.subpixel_shift(o, -0.4 + 0.1 * seed, 0.2)
        for kappa in (10, 100):
            est = registration.register(o, out[f"mov_{k}"], "raw", kappa)
            rows.append((k, 1, kappa, est.dy, est.dx, est.peak_value))
        k += 1
    out["n_pairs"] = k
    out["rows"] = np.array(rows, dtype=np.float64)
    # tie-break pins (test_registration.py:87-100)
    corr = np.zeros((16, 16))
    corr[9, 8] = 1.0
    corr[13, 8] = 1.0
    xps = np.fft.fft2(np.fft.ifftshift(corr))
    c = registration.coarse_shift(xps)
    out["tie_xps"] = xps
    out["tie_est"] = np.array([c.dy, c.dx, c.peak_value])
    np.savez_compressed(OUT / "registration.npz", **out)


def gen_adam():
    out = {}
    cfg = posref.PosRefConfig(step_size=0.3, beta1=0.8, beta2=0.95, max_correction=10)
    buf = posref.AdamBuffers.zeros(3)
    rng = np.random.default_rng(1)
    g_all, d_all = [], []
    for t in range(12):
        g = rng.uniform(-1, 1, (3, 2))
        d = [posref.adam_step(buf, j, tuple(g[j]), cfg) for j in range(3)]
        g_all.append(g)
        d_all.append(d)
    out["g"] = np.array(g_all)
    out["delta"] = np.array(d_all)
    out["m"], out["v"], out["t"] = buf.m, buf.v, buf.t
    pos = np.array([[5.0, 5.0], [9.9, 0.1], [2.5, 7.25]])
    moved = pos.copy()
    for j, dlt in enumerate([(0.25, -0.5), (0.5, -0.5), (-3.0, 4.0)]):
        posref.apply_correction(moved, j, dlt, (0.0, 0.0, 10.0, 10.0))
    out["pos_in"], out["pos_out"] = pos, moved
    np.savez_compressed(OUT / "adam.npz", **out)


def gen_simulate(tmp):
    out = {}
    g, plan, obj, probes, ds = scene(32, (4, 4), 7.0, 8.0, 2, (0.7, 0.3), 1.0, 3)
    out["nominal"], out["true"] = plan.nominal, plan.true_positions
    out["obj"], out["probes"] = obj, np.stack(probes)
    out["patterns"] = ds.patterns
    # config-1 shape digests (BASELINE.json configs[0])
    g1, plan1, obj1, probes1, ds1 = scene(128, (10, 10), 16.0, 30.0, 1, (1.0,), 1.0, 1)
    ds1 = rt32(ds1, tmp / "c1")
    out["c1_digest"] = pattern_digest(ds1.patterns)
    out["c1_positions"] = ds1.positions
    cfg = engine.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5)
    st = engine.initialize(ds1, cfg)
    for _ in range(20):
        engine.sweep(st, ds1, cfg)
    out["c1_error_trace"] = np.array(st.error_trace)
    out["c1_obj_sum"] = np.array([st.obj.sum()])
    out["c1_probe_power"] = np.array([np.sum(np.abs(st.probes[0]) ** 2)])
    np.savez_compressed(OUT / "simulate.npz", **out)


def gen_metrics(tmp):
    """metrics.py:20-64 on a reconstructed scene (object error on the coverage
    mask, position RMSE after the gauge shift)."""
    sys.path.insert(0, str(REF))
    import ptychokit.metrics as metrics
    out = {}
    g, plan, obj, probes, ds = scene(32, (4, 4), 7.0, 8.0, 2, (0.7, 0.3), 1.0, 5)
    cfg = engine.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=2)
    st = engine.initialize(ds, cfg)
    for _ in range(3):
        engine.sweep(st, ds, cfg)
    r0, c0 = st.canvas_origin
    h, w = st.obj.shape
    truth = obj[r0:r0 + h, c0:c0 + w]
    out["recon"], out["truth"] = st.obj, truth
    out["probes"], out["positions"] = np.stack(st.probes), st.positions
    out["canvas_origin"] = np.array(st.canvas_origin)
    for thr in (0.05, 0.3):
        mask = metrics.coverage_mask(st.probes, st.positions, st.obj.shape, st.canvas_origin, thr)
        out[f"mask_{thr}"] = mask
        out[f"object_error_{thr}"] = np.array([metrics.object_error(st.obj, truth, mask)])
    est = plan.true_positions + np.random.default_rng(9).normal(0, 0.3, plan.true_positions.shape) + 2.5
    out["est"], out["true"] = est, plan.true_positions
    out["position_rmse"] = np.array([metrics.position_rmse(est, plan.true_positions)])
    np.savez_compressed(OUT / "metrics.npz", **out)


GENERATORS = {"fields": lambda t: gen_fields(), "visit": gen_visit, "sweeps": gen_sweeps,
              "registration": lambda t: gen_registration(), "adam": lambda t: gen_adam(),
              "simulate": gen_simulate, "metrics": gen_metrics}


def main():
    import tempfile
    only = sys.argv[1:] or list(GENERATORS)
    with tempfile.TemporaryDirectory() as d:
        tmp = Path(d)
        for name in only:
            GENERATORS[name](tmp)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
