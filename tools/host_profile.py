"""cProfile of sweep_replicas host work (R replicas of config 2)."""
import cProfile, pstats, sys
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
R = int(sys.argv[1]) if len(sys.argv) > 1 else 18
cfg = bench.solver_config()
ds = bench.make_dataset()
states = [pk.initialize(ds, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r in range(R)]
for _ in range(2):
    pk.sweep_replicas(states, [ds] * R, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    pk.sweep_replicas(states, [ds] * R, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
