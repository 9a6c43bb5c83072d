"""cProfile of the host side of 18-replica sweeps (where the time between kernels goes)."""
import cProfile, pstats, sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
cfg = bench.solver_config()
R = 18
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(3):
    pk.sweep_replicas(states, dsets, cfgs)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    pk.sweep_replicas(states, dsets, cfgs)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
