"""Cluster vs grid flavour of the line-task sweep: bitwise agreement + timing."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
import paper_2205_04295_b200 as pk

cfg = bench.solver_config()
ds = bench.make_dataset()


def run(R, env, sweeps=3):
    os.environ.update(env)
    states = [pk.initialize(ds, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r in range(R)]
    times = []
    for _ in range(sweeps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pk.sweep_replicas(states, [ds] * R, cfg)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    return states, min(times[1:]) * 1e3


for R in [int(a) for a in sys.argv[1:]] or [16]:
    ref, t_ref = run(R, {"PTY_SWEEP_TILES_MAX": "0", "PTY_CLUSTER": "0"})
    print(f"R={R} grid  {t_ref:.2f} ms  {R*400/t_ref*1e3:.0f} pos/s", flush=True)
    for K in ("16", "8", "4"):
        st, t = run(R, {"PTY_SWEEP_TILES_MAX": "0", "PTY_CLUSTER": K})
        same = all(torch.equal(a.obj, b.obj) and torch.equal(a.probe_stack, b.probe_stack) and
                   a.error_trace == b.error_trace for a, b in zip(st, ref))
        print(f"R={R} cluster{K} {t:.2f} ms {R*400/t*1e3:.0f} pos/s bitwise={same}", flush=True)
    if R <= 8:
        st, t = run(R, {"PTY_SWEEP_TILES_MAX": "8", "PTY_CLUSTER": "16"})
        print(f"R={R} tiles {t:.2f} ms {R*400/t*1e3:.0f} pos/s", flush=True)
