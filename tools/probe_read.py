"""Probe-build timing of the P1 / P4 task internals (CTA 0, thread 0), R replicas."""
import sys, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
import bench
import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import _native
R = int(sys.argv[1])
cfg = bench.solver_config()
dsets = [bench.make_dataset(seed=1 + r) for r in range(R)]
cfgs = bench.replica_configs(cfg, R, 0)
states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
for _ in range(2):
    pk.sweep_replicas(states, dsets, cfgs)
torch.cuda.synchronize()
lib = _native.load()
buf = np.zeros((64, 32), dtype=np.uint64)
assert lib.pty_probe_read(C.c_void_p(buf.ctypes.data)) == 0
b = buf[4:60].astype(np.int64)
names = {0: "P1 start", 1: "o,P0 loaded+om", 2: "team sync", 3: "exit waves (P1,P2 loads)", 4: "3 row FFTs", 5: "team sync", 6: "transposed stores",
         10: "P4 start", 11: "scratch rows staged", 12: "3 inverse FFTs", 13: "team sync", 14: "epilogue"}
for seq in ([0, 1, 2, 3, 4, 5, 6], [10, 11, 12, 13, 14]):
    for a, c in zip(seq, seq[1:]):
        d = (b[:, c] - b[:, a]) / 1e3
        print(f"{names[c]:28s} {np.median(d):7.2f} us (p90 {np.percentile(d, 90):.2f})")
    print()
