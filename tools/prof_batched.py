"""Time batched sweeps: python tools/prof_batched.py <grid> <batch,...> [sweeps]."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 20
batches = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "100").split(",")]
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
bench.GRID = (grid, grid)
ds = bench.make_dataset()
n = ds.n_positions
for b in batches:
    cfg = pk.SolverConfig(**{**bench.solver_config().__dict__, "batch_size": b})
    st = pk.initialize(ds, cfg)
    pk.sweep(st, ds, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(sweeps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); pk.sweep(st, ds, cfg); e.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    print("sweeps", [round(x, 2) for x in ts])
    ms = min(ts)
    print(f"N={n} b={b}: {ms:.2f} ms/sweep  {n/ms*1e3:,.0f} pos/s  roofline {n/ms*1e3*bench.B_POS/6548.5e9:.1%}  err={st.error_trace[-1]:.4f}", flush=True)
