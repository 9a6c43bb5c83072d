"""Per-CTA task-time statistics from the 9-stamp timeline (which CTAs are slow, and is it persistent?).
python tools/tl_cta.py R [sweeps]; PTY_TIMELINE must be set."""
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
act = np.where(tl[0, 1, :] > 0)[0]
tl = tl[:, :, act]
steps = tl.shape[0]
# task time per (step, phase, cta)
task = np.stack([tl[1:steps - 1, 2 * k + 1, :] - tl[1:steps - 1, 2 * k, :] for k in range(4)], axis=1) / 1e3
mean_cta = task.mean(axis=0)                       # (4, ncta)
print("CTAs", len(act), "steps", task.shape[0])
for k in range(4):
    m = mean_cta[k]
    z = (task[:, k, :] - task[:, k, :].mean(axis=1, keepdims=True))
    # persistence: correlation of a CTA's deviation between even and odd steps
    a, b = z[0::2].mean(axis=0), z[1::2].mean(axis=0)
    corr = float(np.corrcoef(a, b)[0, 1])
    print(f"P{k+1}: task mean {m.mean():.2f} us, per-CTA mean min {m.min():.2f} max {m.max():.2f}, "
          f"step-to-step sd {task[:, k, :].std(axis=1).mean():.2f}, persistence corr {corr:.2f}")
    slow = np.argsort(m)[-6:]
    print("   slowest CTAs (block ids):", act[slow].tolist(), np.round(m[slow], 2).tolist())
# CTA b and b+148 share an SM: is the slowness per SM?
sm_pair = {}
for i, bid in enumerate(act):
    sm_pair.setdefault(int(bid) % 148, []).append(i)
smid = _native.timeline().astype(np.int64)[0, 8, act]
print("SM ids of the active CTAs: min", smid.min(), "max", smid.max(), "distinct", len(set(smid.tolist())))
for k in (0, 3):
    m = mean_cta[k]
    order = np.argsort(m)
    print(f"P{k+1} fastest 8 (bid, sm, us):", [(int(act[i]), int(smid[i]), round(float(m[i]), 1)) for i in order[:8]])
    print(f"P{k+1} slowest 8 (bid, sm, us):", [(int(act[i]), int(smid[i]), round(float(m[i]), 1)) for i in order[-8:]])
    # SM-level: CTA count per SM and mean
    per_sm = {}
    for i in range(len(act)):
        per_sm.setdefault(int(smid[i]), []).append(float(m[i]))
    lone = [v[0] for v in per_sm.values() if len(v) == 1]
    pair = [x for v in per_sm.values() if len(v) == 2 for x in v]
    print(f"   CTAs alone on their SM: {len(lone)} mean {np.mean(lone) if lone else float('nan'):.2f}; paired: {len(pair)} mean {np.mean(pair):.2f}")
    # by SM id halves (die guess)
    lo = [float(m[i]) for i in range(len(act)) if smid[i] < 74]
    hi = [float(m[i]) for i in range(len(act)) if smid[i] >= 74]
    print(f"   smid < 74: {np.mean(lo):.2f} us ({len(lo)}), smid >= 74: {np.mean(hi):.2f} us ({len(hi)})")
    # by position within the slot (row quad block)
    pos = np.array([int(a) % 16 for a in act])
    print("   by CTA index within slot:", [round(float(np.mean(m[pos == q])), 1) for q in range(16)])
