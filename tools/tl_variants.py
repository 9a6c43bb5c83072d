"""Per-phase timeline for config variants: python tools/tl_variants.py R"""
import os, sys
sys.path.insert(0, ".")
os.environ.setdefault("PTY_SWEEP_TILES_MAX", "0")
os.environ.setdefault("PTY_TIMELINE", "12")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
R = int(sys.argv[1]) if len(sys.argv) > 1 else 16
ds = bench.make_dataset()
base = bench.solver_config()
for name, kw in [("default", {}), ("no probe update", {"update_probe_modes": False}),
                 ("M=1", {"mode_count": 1})]:
    cfg = pk.SolverConfig(**{**base.__dict__, **kw})
    states = [pk.initialize(ds, pk.SolverConfig(**{**cfg.__dict__, "init_seed": r})) for r in range(R)]
    for _ in range(2):
        pk.sweep_replicas(states, [ds] * R, cfg)
    torch.cuda.synchronize()
    tl = _native.timeline().astype(np.int64)
    ends = tl[:, 1:, :]
    crit = ends.max(axis=2) - np.concatenate([tl[:, 0, :].max(axis=1)[:, None], ends.max(axis=2)[:, :3]], axis=1)
    print(name, np.round(np.median(crit[1:10], axis=0) / 1e3, 2), flush=True)
