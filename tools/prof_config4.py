"""Config 4 (512^2 x 5 modes, Fresnel, posref XCORR_A kappa=10) with R replicas: python tools/prof_config4.py R [sweeps] [--noposref]."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
R = int(sys.argv[1]); sweeps = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else 2
c = bench.CONFIGS["config4"]
w, m = c["W"], c["M"]
geom = pk.Geometry.create(c["lam"], 0.75, 20e-6, w)
plan = pk.make_scan(c["grid"], c["step"], 1.0, seed=1)
obj = pk.make_object(pk.canvas_shape_for(plan, w), "spokes", seed=1)
probes = pk.make_probe(pk.ProbeSpec(m, c["powers"], "disk", c["radius"]), geom)
ds = pk.synthesize(obj, probes, plan, geom, noise="none", seed=1, propagator=c["propagator"])
ds.patterns = ds.patterns.astype(np.float32)
ds.positions = ds.positions + np.random.default_rng(42).uniform(-2, 2, ds.positions.shape)
posref = None if "--noposref" in sys.argv else pk.PosRefConfig(sensor="XCORR_A", kappa=10, warmup_iterations=0)
cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=m, position_order="shuffled",
                      posref=posref, propagator=c["propagator"])
cfgs = bench.replica_configs(cfg, R, 0)
sts = [pk.initialize(ds, cc) for cc in cfgs]
for _ in range(sweeps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pk.sweep_replicas(sts, [ds] * R, cfgs); b.record(); torch.cuda.synchronize()
    print(f"config4 R={R} posref={posref is not None} sweep {a.elapsed_time(b):.1f} ms -> {R*1600/a.elapsed_time(b)*1e3:,.0f} pos/s", flush=True)
