"""R replicas (own datasets) for ncu: python tools/prof_tl.py R [sweeps]."""
import sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
R = int(sys.argv[1]); sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(sweeps):
    pk.sweep_replicas(states, dsets, cfgs)
torch.cuda.synchronize()
print("done", states[0].error_trace[-1])
