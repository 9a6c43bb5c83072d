import os, sys, traceback
sys.path[:0] = [".", "tests"]
import torch, torch.distributed as dist
import paper_2205_04295_b200 as pk
from conftest import golden
from test_gpu_parity import make_ds, pkg_cfg
from test_oracle_golden import cfg_from_repr
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
torch.cuda.set_device(0)
try:
    g = golden("sweep_posref_a")
    c = pkg_cfg(cfg_from_repr(str(g["cfg_repr"])), "fp64")
    cfg = pk.SolverConfig(**{**c.__dict__, "batch_size": 6})
    ds = make_ds(g["patterns"], g["positions_in"], g["window"])
    st = pk.initialize(ds, cfg)
    for k in range(int(g["sweeps"])):
        pk.sweep(st, ds, cfg, group=dist.group.WORLD)
        print(rank, "sweep", k, st.error_trace[-1], st.positions[:3].tolist(), flush=True)
except Exception:
    traceback.print_exc()
    sys.stdout.flush()
    os._exit(1)
