"""Sweep timing for given replica counts and env flavours: python tools/quick_time.py R [R...]"""
import os, sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
cfg = bench.solver_config()
ds = bench.make_dataset()
for R in [int(a) for a in sys.argv[1:]] or [16]:
    states = [pk.initialize(ds, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r in range(R)]
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        pk.sweep_replicas(states, [ds] * R, cfg)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    t = min(ts[1:]) * 1e3
    print(f"R={R} {t:.2f} ms/sweep {R*ds.n_positions/t*1e3:.0f} pos/s err={states[0].error_trace[-1]:.6f}", flush=True)
