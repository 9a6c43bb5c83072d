"""Per-phase task time vs barrier wait from the 9-stamp sweep timeline.

python tools/tl_phases.py R [sweeps] [--same-data]: R replicas of config 2 (own
datasets unless --same-data), PTY_TIMELINE must be set (steps to record)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native

R = int(sys.argv[1])
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 2
same = "--same-data" in sys.argv
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 if same else 1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(sweeps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); pk.sweep_replicas(states, dsets, cfgs); b.record(); torch.cuda.synchronize()
    print(f"R={R} sweep {a.elapsed_time(b):.2f} ms  -> {R*400/a.elapsed_time(b)*1e3:,.0f} pos/s", flush=True)
tl = _native.timeline().astype(np.int64)          # (steps, 9, grid)
act = tl[0, 1, :] > 0                              # CTAs that did work
tl = tl[:, :, act]
steps = tl.shape[0]
task = np.zeros(4); wait = np.zeros(4); crit = np.zeros(4); tmax = np.zeros(4)
for s_ in range(2, steps - 1):   # step 1 stamp 8 carries the virtual CTA index
    for k in range(4):
        start = tl[s_, 2 * k, :]                  # barrier exit of the previous phase (k=0: step start)
        end = tl[s_, 2 * k + 1, :]
        ext = tl[s_, 2 * k + 2, :]
        task[k] += np.mean(end - start)
        tmax[k] += np.mean(np.max(end - start))
        wait[k] += np.mean(ext - end)
        crit[k] += np.max(ext) - np.max(start)
n = steps - 3
print("phase        P1     P2     P3     P4   (us, mean over CTAs and steps)")
print("task mean ", np.round(task / n / 1e3, 2))
print("task max  ", np.round(tmax / n / 1e3, 2))
print("wait mean ", np.round(wait / n / 1e3, 2))
print("crit path ", np.round(crit / n / 1e3, 2), " step", round(float(np.sum(crit / n / 1e3)), 2))
