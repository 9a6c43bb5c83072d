"""The engine's multi-rank batched sweep (sweep_batched with a process group)
on ONE GPU: two processes share the device, each runs its share of every batch
through the CUDA kernels and the update terms are all-reduced with gloo (host
copies; no kernel waits on another).  Result == the single-process batched
sweep of the same batches (the NCCL path on 2-8 GPUs runs the same code:
spatial shares, halo rows to their owner, owned rows all-gathered,
partition.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import golden

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, q, name):
    import torch.distributed as dist
    import paper_2205_04295_b200 as pk
    from test_gpu_parity import make_ds, pkg_cfg
    from test_oracle_golden import cfg_from_repr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = golden(f"sweep_{name}")
    c = pkg_cfg(cfg_from_repr(str(g["cfg_repr"])), "fp64")
    cfg = pk.SolverConfig(**{**c.__dict__, "batch_size": 6})
    ds = make_ds(g["patterns"], g["positions_in"], g["window"])
    st = pk.initialize(ds, cfg)
    for _ in range(max(2, int(g["sweeps"]))):
        pk.sweep(st, ds, cfg, group=dist.group.WORLD if world > 1 else None)
    q.put((rank, st.obj.cpu().numpy(), st.probe_stack.cpu().numpy(), list(st.error_trace),
           st.positions.cpu().numpy(), None if st.adam is None else st.adam.t.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _spawn(world, name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q, name)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=300) for _ in range(world)), key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return outs


@pytest.mark.parametrize("name", ["rpie", "posref_a", "posref_b"])
def test_two_rank_batched_sweep_matches_one_rank(gpu, name):
    one = _spawn(1, name)[0]
    twos = _spawn(2, name)
    for two in twos:                      # every rank holds the same state
        scale = np.linalg.norm(one[1])
        assert np.linalg.norm(two[1] - one[1]) / scale < 1e-12
        assert np.linalg.norm(two[2] - one[2]) / np.linalg.norm(one[2]) < 1e-12
        np.testing.assert_allclose(two[3], one[3], rtol=1e-12)
        np.testing.assert_allclose(two[4], one[4], rtol=0, atol=1e-9)
        if one[5] is not None:
            np.testing.assert_array_equal(two[5], one[5])
    np.testing.assert_array_equal(twos[0][4], twos[1][4])


def test_two_rank_batched_sweep_reruns_bitwise(gpu):
    """The 2-rank decomposition is deterministic: two runs are bit-identical
    (fixed shares, fixed halo order, fixed reduction order)."""
    a = _spawn(2, "posref_a")
    b = _spawn(2, "posref_a")
    for x, y in zip(a, b):
        assert np.array_equal(x[1], y[1]) and np.array_equal(x[2], y[2])
        assert x[3] == y[3]
        assert np.array_equal(x[4], y[4])
