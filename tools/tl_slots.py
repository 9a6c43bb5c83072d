"""Per-slot view of the 9-stamp timeline: which slots are slow, and how the two
slots sharing an SM set are phased against each other.
python tools/tl_slots.py R [sweeps]; PTY_TIMELINE must be set (>= 3 steps)."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
R = int(sys.argv[1]); sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(sweeps):
    pk.sweep_replicas(states, dsets, cfgs)
torch.cuda.synchronize()
tl = _native.timeline().astype(np.int64)
vcta = tl[1, 8, :].copy()
act = np.where(tl[0, 1, :] > 0)[0]
steps = tl.shape[0]
cps = 16
slot = vcta[act] // cps
S = int(slot.max()) + 1
spp = S // 2
rows = []
for s in range(S):
    ids = act[slot == s]
    t = tl[2:steps - 1, :, ids]                      # (steps, 9, ctas)
    period = np.median(np.diff(t[:, 0, :].min(axis=1)))
    ph = [np.mean(t[:, 2 * k + 1, :].max(axis=1) - t[:, 2 * k, :].min(axis=1)) for k in range(4)]
    rows.append((s, len(ids), period / 1e3, [round(x / 1e3, 2) for x in ph]))
start = {s: tl[2:steps - 1, 0, act[slot == s]].min(axis=1) for s in range(S)}
for s, n, per, ph in rows:
    partner = s + spp if s < spp else s - spp
    off = ""
    if partner in start:
        d = (start[s] - start[partner]) / 1e3
        off = f" start - partner start: median {np.median(d):7.2f} us (mod period {np.median(d) % per:5.2f})"
    print(f"slot {s:2d} ({n} CTAs): step {per:6.2f} us  phase spans {ph}{off}")
