"""Multi-rank decomposition of the batched extension, on CPU with gloo
(world_size 2): every rank computes the update terms of its contiguous share
of each batch (engine.batch_slice), the terms are all-reduced (sum) and every
rank applies them -- the same steps engine.sweep_batched runs with NCCL.  The
result must equal the single-rank batched sweep (oracle/batched.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden
from oracle import batched, rpie
from paper_2205_04295_b200.engine import batch_slice
from test_oracle_golden import cfg_from_repr


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce_complex(a):
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).copy())
    dist.all_reduce(t)
    return t.numpy().view(np.complex128).reshape(a.shape)


def _allreduce_real(a):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).copy())
    dist.all_reduce(t)
    return t.numpy()


def _worker(rank, world, port, batch, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("sweep_rpie")
    cfg = cfg_from_repr(str(g["cfg_repr"]))
    w = int(g["window"])
    pats = g["patterns"].astype(np.float64)
    st = rpie.initialize(pats, g["positions_in"], w, cfg)
    for _ in range(2):
        order = rpie.visit_order(len(pats), cfg.position_order, cfg.shuffle_seed, st.iteration)
        num = den = 0.0
        for s in range(0, len(pats), batch):
            ids = order[s:s + batch]
            lo, hi = batch_slice(len(ids), rank, world)
            t = batched.contrib(st, pats, w, cfg, ids[lo:hi])
            t.onum = _allreduce_complex(t.onum)
            t.oden = _allreduce_real(t.oden)
            t.pnum = [_allreduce_complex(p) for p in t.pnum]
            t.pden = _allreduce_real(t.pden)
            e = _allreduce_real(np.array([t.err_num, t.err_den]))
            num += e[0]
            den += e[1]
            batched.apply(st, cfg, t)
        st.error_trace.append(num / den)
    if rank == 0:
        out_q.put((st.obj, np.stack(st.probes), st.error_trace))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [4, 7])
def test_two_rank_batched_sweep_equals_single_rank(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    obj, probes, trace = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = golden("sweep_rpie")
    cfg = cfg_from_repr(str(g["cfg_repr"]))
    w = int(g["window"])
    pats = g["patterns"].astype(np.float64)
    ref = rpie.initialize(pats, g["positions_in"], w, cfg)
    for _ in range(2):
        batched.sweep_batched(ref, pats, w, cfg, batch)
    np.testing.assert_allclose(obj, ref.obj, rtol=0, atol=1e-13)
    np.testing.assert_allclose(probes, np.stack(ref.probes), rtol=0, atol=1e-13)
    np.testing.assert_allclose(trace, ref.error_trace, rtol=1e-12)


def test_batch_slices_partition_the_batch():
    for n in (1, 5, 16, 401):
        for world in (1, 2, 3, 8):
            spans = [batch_slice(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
