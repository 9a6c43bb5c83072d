import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2205_04295_b200 as pk
from oracle import rpie, registration as oreg
from conftest import golden

def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))

g = golden("registration")
for pair, weighting, kappa, dy, dx, peak in g["rows"]:
    k = int(pair)
    est = pk.register(g[f"ref_{k}"], g[f"mov_{k}"], ["phase", "raw"][int(weighting)], int(kappa))
    if abs(est.peak_value - peak) > 1e-9 * abs(peak):
        print("REG", k, int(weighting), int(kappa), est, peak)

geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 128)
plan = pk.make_scan((10, 10), 16.0, 1.0, seed=1)
obj = pk.make_object(pk.canvas_shape_for(plan, 128), "spokes", seed=1)
probes = pk.make_probe(pk.ProbeSpec(1, (1.0,), "disk", 30.0), geom)
ds = pk.synthesize(obj, probes, plan, geom)
ds.patterns = ds.patterns.astype(np.float32).astype(np.float64)
cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, precision="fp64")
st = pk.initialize(ds, cfg)
ost = rpie.initialize(ds.patterns, ds.positions, 128, cfg)
print("init probe", rel(st.probe_stack.cpu().numpy()[0], ost.probes[0]), st.canvas_origin, ost.canvas_origin, st.obj.shape, ost.obj.shape)
for it in range(6):
    pk.sweep(st, ds, cfg)
    rpie.sweep(ost, ds.patterns, 128, cfg)
    print(it, "obj", rel(st.obj.cpu().numpy(), ost.obj), "probe", rel(st.probe_stack.cpu().numpy()[0], ost.probes[0]), st.error_trace[-1], ost.error_trace[-1])
# single visit at W=128 M=1 from the same state
t = pk._native.torch()
