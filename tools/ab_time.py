"""A/B sweep timing that runs in any tree of this repo: R replicas of config 2,
each its own dataset and visit order (passed as orders=), kernel time per sweep.
python tools/ab_time.py R [sweeps]"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200.engine import visit_order
R = int(sys.argv[1]); sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
states = [pk.initialize(d, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r, d in enumerate(dsets)]
ts = []
for it in range(sweeps):
    orders = [visit_order(400, pk.SolverConfig(**{**cfg.__dict__, "shuffle_seed": r}), st.iteration)
              for r, st in enumerate(states)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pk.sweep_replicas(states, dsets, cfg, orders=orders); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
best = sorted(ts[2:])[len(ts[2:]) // 2]
print(f"{os.environ.get('TAG','')} R={R} median {best:.2f} ms  {R*400/best*1e3:,.0f} pos/s  all={[round(x,2) for x in ts]}", flush=True)
