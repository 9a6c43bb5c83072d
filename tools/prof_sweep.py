"""Run a few config-2 sweeps with R replicas (for ncu / timeline runs)."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.solver_config()
ds = bench.make_dataset()
states = [pk.initialize(ds, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r in range(R)]
for _ in range(sweeps):
    t0 = time.perf_counter()
    pk.sweep_replicas(states, [ds] * R, cfg)
    torch.cuda.synchronize()
    print(f"R={R} sweep {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
if "--barrier" in sys.argv:
    for c in (148, 74, 32):
        print("barrier ns", c, _native.barrier_bench(20000, c))
if "--timeline" in sys.argv:
    import os, numpy as np
    tl = _native.timeline().astype(np.int64)
    if tl.size:
        start = tl[:, 0, :].min(axis=1)                 # step start (first CTA)
        ends = tl[:, 1:, :]                              # per-CTA phase ends
        prev = np.concatenate([start[:, None], ends.max(axis=2)[:, :3]], axis=1)
        # barrier exit ~ next phase's first stamp; phase critical path = max end - previous phase exit
        steps = tl.shape[0]
        crit = ends.max(axis=2) - np.concatenate([tl[:, 0, :].max(axis=1)[:, None], ends.max(axis=2)[:, :3]], axis=1)
        nxt = np.concatenate([tl[1:, 0, :].max(axis=1), [0]])
        print("per-step us: P1 P2 P3 P4 (max CTA end - previous max end); step total")
        for s_ in range(1, min(steps - 1, 8)):
            tot = (tl[s_ + 1, 0, :].max() - tl[s_, 0, :].max()) / 1e3
            print(s_, np.round(crit[s_] / 1e3, 2), round(tot, 2))
        # mean CTA-completion spread per phase
        spread = (ends.max(axis=2) - ends.min(axis=2)).mean(axis=0) / 1e3
        print("mean (max-min) CTA end spread per phase us:", np.round(spread, 2))
