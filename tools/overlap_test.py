"""H2D (copy stream) concurrently with the sweep (main stream): do they overlap?"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
R = 18
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
hosts = [torch.from_numpy(np.ascontiguousarray(d.patterns, np.float32)).pin_memory() for d in dsets]
devs = [torch.empty(h.shape, dtype=torch.float32, device="cuda") for h in hosts]
cs = torch.cuda.Stream()
for _ in range(2):
    pk.sweep_replicas(states, dsets, cfgs)
def copy_only():
    with torch.cuda.stream(cs):
        for d, h in zip(devs, hosts): d.copy_(h, non_blocking=True)
    cs.synchronize()
def ev(): return torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); t = time.perf_counter(); copy_only(); print("H2D alone %.1f ms" % (1e3 * (time.perf_counter() - t)))
torch.cuda.synchronize(); t = time.perf_counter(); pk.sweep_replicas(states, dsets, cfgs); torch.cuda.synchronize(); print("sweep alone %.1f ms" % (1e3 * (time.perf_counter() - t)))
for k in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    a0, a1, b0, b1 = ev(), ev(), ev(), ev()
    with torch.cuda.stream(cs):
        a0.record(cs)
        for d, h in zip(devs, hosts): d.copy_(h, non_blocking=True)
        a1.record(cs)
    b0.record()
    pk.sweep_replicas(states, dsets, cfgs)
    b1.record()
    torch.cuda.synchronize()
    print("concurrent: wall %.1f ms, copy %.1f ms, sweep %.1f ms, copy start->sweep start %.1f ms" % (
        1e3 * (time.perf_counter() - t), a0.elapsed_time(a1), b0.elapsed_time(b1), a0.elapsed_time(b0)))
