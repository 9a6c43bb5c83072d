"""Multi-rank decomposition of the batched extension, on CPU with gloo
(world_size 2): every batch is split spatially (paper_2205_04295_b200/
partition.py -- the same host logic engine.sweep_batched runs with NCCL):
each rank computes the update terms of its row-sorted share, halo rows are
sent point-to-point to their owner, which adds them in rank order, the owned
rows are all-gathered and the probe terms all-reduced; every rank applies the
identical update.  The result must equal the single-rank batched sweep
(oracle/batched.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden
from oracle import batched, rpie
from paper_2205_04295_b200.partition import (batch_slice, halo_transfers, ownership, rank_shares,
                                             row_bands)
from test_oracle_golden import cfg_from_repr


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a).view(np.float64).copy())
    dist.all_reduce(t)
    return t.numpy().view(a.dtype).reshape(a.shape)


def _exchange_rows(acc, owns, xfers, rank, world):
    """partition.py exchange on a (rows, cols) float64 accumulator."""
    ops, recvs = [], []
    for src, dst, a, b in xfers:
        if src == rank:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(acc[a:b].copy()), dst))
        elif dst == rank:
            buf = torch.empty((b - a, acc.shape[1]), dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, buf, src))
            recvs.append((a, b, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for a, b, buf in recvs:
        acc[a:b] += buf.numpy()
    R = max(hi - lo for lo, hi in owns)
    if R == 0:
        return acc
    lo, hi = owns[rank]
    send = torch.zeros((R, acc.shape[1]), dtype=torch.float64)
    send[:hi - lo] = torch.from_numpy(acc[lo:hi])
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send)
    for q, (qlo, qhi) in enumerate(owns):
        if q != rank and qhi > qlo:
            acc[qlo:qhi] = parts[q][:qhi - qlo].numpy()
    return acc


def _worker(rank, world, port, batch, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("sweep_rpie")
    cfg = cfg_from_repr(str(g["cfg_repr"]))
    w = int(g["window"])
    pats = g["patterns"].astype(np.float64)
    st = rpie.initialize(pats, g["positions_in"], w, cfg)
    h, wc = st.obj.shape
    for _ in range(2):
        order = rpie.visit_order(len(pats), cfg.position_order, cfg.shuffle_seed, st.iteration)
        rows_all = np.array([rpie.anchor(p)[0] for p in st.positions]) - st.canvas_origin[0]
        num = den = 0.0
        for s in range(0, len(pats), batch):
            ids = order[s:s + batch]
            rows = rows_all[ids]
            shares = rank_shares(rows, world)
            bands = row_bands(rows, shares, w, h)
            owns = ownership(bands)
            xf = halo_transfers(bands, owns)
            t = batched.contrib(st, pats, w, cfg, ids[shares[rank]])
            # the object terms as [row][re, im, den][col] (the engine's layout)
            acc = np.stack([t.onum.real, t.onum.imag, t.oden], axis=1).reshape(h, 3 * wc)
            acc = _exchange_rows(acc, owns, xf, rank, world).reshape(h, 3, wc)
            t.onum = acc[:, 0] + 1j * acc[:, 1]
            t.oden = acc[:, 2].copy()
            t.pnum = [_allreduce(p) for p in t.pnum]
            t.pden = _allreduce(t.pden)
            e = _allreduce(np.array([t.err_num, t.err_den]))
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


def test_spatial_partition_covers_every_row_once():
    """rank_shares / row_bands / ownership / halo_transfers: every batch
    position is on exactly one rank, the owned ranges tile the batch's band,
    and every accumulator row a rank computed either is its own or is sent to
    the one rank that owns it."""
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        for n in (1, 3, 40, 400):
            rows = rng.integers(0, 500, n)
            shares = rank_shares(rows, world)
            assert sorted(np.concatenate(shares).tolist()) == list(range(n))
            bands = row_bands(rows, shares, 64, 600)
            owns = ownership(bands)
            xf = halo_transfers(bands, owns)
            live = [o for o in owns if o[1] > o[0]]
            assert live[0][0] == int(rows.min()) and live[-1][1] == min(600, int(rows.max()) + 64)
            for (a, b), (c, d) in zip(live, live[1:]):
                assert b == c
            for r, (lo, hi) in enumerate(bands):
                for row in range(lo, hi):
                    owner = [q for q, (olo, ohi) in enumerate(owns) if olo <= row < ohi]
                    assert len(owner) == 1
                    if owner[0] != r:
                        assert any(src == r and dst == owner[0] and a <= row < b for src, dst, a, b in xf)


def test_batch_slices_partition_the_batch():
    for n in (1, 5, 16, 401):
        for world in (1, 2, 3, 8):
            spans = [batch_slice(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
