"""Config 3 in replica mode (posref XCORR_A kappa=10 engaged), R replicas, for
launch lists: python tools/prof_posref.py R [sweeps]."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
R = int(sys.argv[1]); sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dsets = []
for r in range(R):
    d = bench.make_dataset(seed=1 + r)
    d.positions = d.positions + np.random.default_rng(42 + r).uniform(-2, 2, d.positions.shape)
    dsets.append(d)
cfg = pk.SolverConfig(**{**bench.solver_config().__dict__,
                         "posref": pk.PosRefConfig(sensor="XCORR_A", kappa=10, warmup_iterations=0)})
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(sweeps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pk.sweep_replicas(states, dsets, cfgs); b.record(); torch.cuda.synchronize()
    print(f"R={R} posref sweep {a.elapsed_time(b):.2f} ms", flush=True)
