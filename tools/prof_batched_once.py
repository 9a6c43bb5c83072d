"""One batched sweep of config 5 (for ncu launch lists): python tools/prof_batched_once.py [batch]."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
bench.GRID = (80, 80)
ds = bench.make_dataset(seed=5)
cfg = pk.SolverConfig(**{**bench.solver_config().__dict__, "batch_size": b})
st = pk.initialize(ds, cfg)
pk.sweep(st, ds, cfg)
torch.cuda.synchronize()
print("done", st.error_trace[-1])
