"""Per-SM task times from the 9-stamp timeline, for several replica counts in
one process: is a CTA's persistent slowness a property of its SM?
python tools/tl_sm.py R1,R2,...; PTY_TIMELINE must be set."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
cfg = bench.solver_config()
res = {}
for R in [int(x) for x in sys.argv[1].split(",")]:
    dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
    cfgs = bench.replica_configs(cfg, R, 0)
    states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
    for _ in range(2):
        pk.sweep_replicas(states, dsets, cfgs)
    torch.cuda.synchronize()
    tl = _native.timeline().astype(np.int64)
    act = np.where(tl[0, 1, :] > 0)[0]
    smid = tl[0, 8, act]
    vcta = tl[1, 8, act]
    t = tl[2:-1][:, :, act]
    task = np.stack([(t[:, 2 * k + 1] - t[:, 2 * k]).mean(axis=0) for k in range(4)])  # (4, ncta)
    per_sm = np.full((4, 148), np.nan)
    for k in range(4):
        for sm in range(148):
            sel = smid == sm
            if sel.any():
                per_sm[k, sm] = task[k, sel].mean()
    res[R] = per_sm
    tot = np.nansum(per_sm, axis=0)
    print(f"R={R}: per-SM total task time over phases: min {np.nanmin(np.where(tot > 0, tot, np.nan)):.1f} "
          f"median {np.nanmedian(np.where(tot > 0, tot, np.nan)):.1f} max {np.nanmax(tot):.1f} us")
    # by rq (vcta % 16)
    rq = vcta % 16
    print("   P1 by rq:", [round(float(task[0, rq == q].mean()), 1) for q in range(16)])
    print("   P4 by rq:", [round(float(task[3, rq == q].mean()), 1) for q in range(16)])
    sl = vcta // 16
    print("   P4 by slot:", [round(float(task[3, sl == q].mean()), 1) for q in range(int(sl.max()) + 1)])
Rs = list(res)
for i in range(len(Rs)):
    for j in range(i + 1, len(Rs)):
        a, b = res[Rs[i]], res[Rs[j]]
        for k in range(4):
            ok = ~np.isnan(a[k]) & ~np.isnan(b[k])
            if ok.sum() > 10:
                print(f"corr per-SM P{k+1} R={Rs[i]} vs R={Rs[j]}: {np.corrcoef(a[k, ok], b[k, ok])[0, 1]:.2f} (n={ok.sum()})")
np.save("gpurun_out/tl_sm.npy", np.stack([res[r] for r in Rs]))
