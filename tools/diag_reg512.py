import sys, numpy as np
sys.path[:0] = [".", "tests"]
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
from oracle import registration as oreg
import torch
for W in (256, 512):
    geom = pk.Geometry.create(8.29e-10, 0.75, 20e-6, W)
    plan = pk.make_scan((3, 3), W / 8, 1.0, seed=4)
    obj = pk.make_object(pk.canvas_shape_for(plan, W), "spokes", seed=4)
    probes = pk.make_probe(pk.ProbeSpec(1, (1.0,), "disk", W * 0.23), geom)
    ds = pk.synthesize(obj, probes, plan, geom)
    cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=1,
                          precision=sys.argv[1], posref=pk.PosRefConfig(kappa=10, warmup_iterations=0))
    st = pk.initialize(ds, cfg)
    saved = {}
    orig = pk.engine._refine_positions
    def spy(st_, pc, n_, w_):
        saved["s"] = st_.buffer("stage", (n_, 2, w_, w_), st_.obj.dtype).clone()
        return orig(st_, pc, n_, w_)
    pk.engine._refine_positions = spy
    pk.sweep(st, ds, cfg)
    pk.engine._refine_positions = orig
    n = ds.n_positions
    stage = saved["s"].clone()
    dy = st.buffer("reg_dy", (n,), torch.float64); dx = st.buffer("reg_dx", (n,), torch.float64)
    peak = st.buffer("reg_peak", (n,), torch.float64); ok = st.buffer("reg_ok", (n,), torch.int32)
    s = saved['s'].cpu().numpy()
    for kap in (1, 2, 10):
        stage = saved["s"].clone()
        _native.register_batch(stage, W, n, 1, kap, dy, dx, peak, ok)
        for j in range(n):
            try:
                e = oreg.register(s[j, 0], s[j, 1], "raw", kap)
                o = (e.dx, e.dy, e.peak_value)
            except oreg.Degenerate:
                o = None
            print(W, kap, j, "gpu", float(dx[j]), float(dy[j]), float(peak[j]), int(ok[j]), "oracle", o, flush=True)
