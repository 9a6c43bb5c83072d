"""Host (numpy) scene builder for CPU-side tests: the package's scene
generators (simulate.make_scan/make_probe/make_object, pinned to the reference
by test_host_cpu.py) plus a numpy restatement of simulate.synthesize
(simulate.py:157-198) for noiseless data."""

import numpy as np

import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import simulate as sim
from oracle import rpie


def host_scene(window, grid, step, radius, modes, powers, jitter=1.0, seed=1, kind="spokes"):
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, window)
    plan = sim.make_scan(grid, step, jitter, seed=seed)
    obj = sim.make_object(sim.canvas_shape_for(plan, window), kind, seed=seed)
    probes = sim.make_probe(sim.ProbeSpec(modes, powers, "disk", radius), geom)
    fy = np.fft.fftfreq(window)[:, None]
    fx = np.fft.fftfreq(window)[None, :]
    pats = np.empty((len(plan.true_positions), window, window))
    for j, (x, y) in enumerate(plan.true_positions):
        ar, ac = int(round(float(y))), int(round(float(x)))
        view = obj[ar:ar + window, ac:ac + window]
        ry, rx = y - ar, x - ac
        if rx != 0.0 or ry != 0.0:
            view = np.fft.ifft2(np.fft.fft2(view) * np.exp(-2j * np.pi * (fy * -ry + fx * -rx)))
        pats[j] = sum(np.abs(rpie.centered_fft2(p * view)) ** 2 for p in probes)
    pats = pats.astype(np.float32).astype(np.float64)      # on-disk precision
    ds = pk.PtychoDataset(patterns=pats, positions=plan.nominal.copy(), geometry=geom)
    return ds, obj, probes, plan
