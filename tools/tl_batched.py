"""Per-phase task / wait times of the batched line-task flavour (config 5, one
batch of b positions): python tools/tl_batched.py [b]; PTY_TIMELINE must be set."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
b = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
bench.GRID = (80, 80)
ds = bench.make_dataset(seed=5)
cfg = pk.SolverConfig(**{**bench.solver_config().__dict__, "batch_size": b})
st = pk.initialize(ds, cfg)
pk.sweep(st, ds, cfg)
torch.cuda.synchronize()
tl = _native.timeline().astype(np.int64)
act = tl[0, 1, :] > 0
tl = tl[:, :, act]
n = tl.shape[0]
task = np.zeros(4); wait = np.zeros(4)
for s_ in range(1, n - 1):
    for k in range(4):
        start = tl[s_, 2 * k, :]; end = tl[s_, 2 * k + 1, :]; ext = tl[s_, 2 * k + 2, :] if k < 3 else tl[s_ + 1, 0, :]
        task[k] += np.mean(end - start); wait[k] += np.mean(ext - end)
print("phase        P1     P2     P3     P4   (us, mean over CTAs and steps; P4 wait = gap to next step)")
print("task mean ", np.round(task / (n - 2) / 1e3, 2))
print("wait mean ", np.round(wait / (n - 2) / 1e3, 2))
per = np.median(np.diff(tl[:, 0, :], axis=0)) / 1e3
print("step period (median over CTAs)", round(float(per), 2), "us")
