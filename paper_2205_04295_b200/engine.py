"""Multi-mode rPIE reconstruction engine on the B200 (drop-in for ptychokit.engine).

Same public surface as /root/reference/pkg/src/ptychokit/engine.py:
``SolverConfig`` (engine.py:25-50, same fields/defaults/validation plus the
``precision`` extension), ``ReconState`` (engine.py:53-66), ``initialize``
(engine.py:73-101), ``sweep`` (engine.py:173-243) and ``run``
(engine.py:246-260).  The state lives in HBM as torch tensors; one ``sweep``
is one cooperative CUDA launch over every position (pty_sweep), followed, when
position refinement is engaged, by one batched registration launch over the
staged (o_j, o'_j) crops and one float64 Adam launch (posref.py:87-113).

What stays on the host (exactly as in the reference, and cheap): the visit
permutation default_rng([shuffle_seed, iteration]) (engine.py:177-181), the
canvas bounding box from Python round() anchors (engine.py:76-81) and the
default_rng([init_seed, p]) noise of extra probe modes (engine.py:87-90).

Deviations: windows must be powers of two in
[16, 512]; negative intensities raise DataError when the dataset is first
uploaded rather than at the offending visit; out-of-canvas anchors raise
BoundsError before any visit of the sweep is applied.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native
from .dataio import read_checkpoint, write_checkpoint
from .errors import ParameterError, ShapeError, raise_for_status
from .fields import check_window
from .posref import AdamBuffers, PosRefConfig

TINY = np.finfo(float).tiny


@dataclass(frozen=True)
class SolverConfig:
    alpha_obj: float = 0.9
    alpha_probe: float = 0.9
    beta: float = 1.0                 # probe-update regularisation, (0, 1]
    gamma: float = 1.0                # object-update regularisation, (0, 1]
    mode_count: int = 1
    iterations: int = 100
    position_order: str = "shuffled"  # fixed | shuffled
    shuffle_seed: int = 0
    init_seed: int = 0
    epsilon_rel: float = 1e-12        # denominator guard, relative to its max
    ortho_interval: int = 0           # Gram-Schmidt probe modes every k iters; 0 = off
    update_probe_modes: bool = True
    posref: PosRefConfig | None = None
    track_modulus_error: bool = False
    precision: str = "fp32"           # B200 extension: fp32 (complex64) | fp64 (complex128)
    batch_size: int = 1               # B200 extension: >1 = batched semi-parallel update
    propagator: str = "farfield"      # B200 extension: farfield | fresnel (single-FFT Fresnel regime)
    subpixel_gather: bool = False     # B200 extension: crops at the float position (residual Fourier shift)

    def __post_init__(self) -> None:
        if not (0 <= self.alpha_obj <= 1 and 0 <= self.alpha_probe <= 1):
            raise ParameterError("update rates must lie in [0, 1]")
        if not (0 < self.beta <= 1 and 0 < self.gamma <= 1):
            raise ParameterError("beta and gamma must lie in (0, 1]")
        if self.position_order not in ("fixed", "shuffled"):
            raise ParameterError(f"unknown position order {self.position_order!r}")
        if self.mode_count < 1:
            raise ParameterError("mode_count must be >= 1")
        if self.mode_count > 8:
            raise ParameterError("mode_count must be <= 8 on the B200 path")
        if self.precision not in ("fp32", "fp64"):
            raise ParameterError(f"precision must be 'fp32' or 'fp64', got {self.precision!r}")
        if self.batch_size < 1:
            raise ParameterError("batch_size must be >= 1")
        if self.propagator not in ("farfield", "fresnel"):
            raise ParameterError(f"propagator must be 'farfield' or 'fresnel', got {self.propagator!r}")
        if self.subpixel_gather and self.batch_size > 1:
            raise ParameterError("subpixel_gather is a sequential-sweep extension (batch_size must be 1)")
        if self.subpixel_gather and self.track_modulus_error:
            raise ParameterError("track_modulus_error is not available with subpixel_gather")


class ReconState:
    """Reconstruction state resident on the GPU (engine.py:53-66).

    ``obj`` (H, Wc) and the probe stack (M, W, W) are complex64/complex128
    CUDA tensors; ``probes`` is a list view over the stack (assigning a list
    restacks it); ``positions`` is an (N, 2) float64 CUDA tensor.

    With the Fresnel propagator the stack holds the probes in the kernels'
    frame, P * Q (Q = fresnel_chirp); ``probes`` returns P = stack * conj(Q)."""

    def __init__(self, obj, probes, positions, canvas_origin, adam=None,
                 error_trace=None, modulus_error_trace=None, seconds_per_iteration=None,
                 frame_chirp=None):
        t = _native.torch()
        self.frame_chirp = frame_chirp
        self.obj = obj
        self.probe_stack = probes if isinstance(probes, t.Tensor) else t.stack(list(probes))
        self.positions = positions
        self.canvas_origin = (int(canvas_origin[0]), int(canvas_origin[1]))
        self.adam = adam
        self.error_trace = list(error_trace or [])
        self.modulus_error_trace = list(modulus_error_trace or [])
        self.seconds_per_iteration = list(seconds_per_iteration or [])
        self._buf = {}

    @property
    def probes(self):
        if self.frame_chirp is not None:
            return list((self.probe_stack * self.frame_chirp.conj()).unbind(0))
        return list(self.probe_stack.unbind(0))

    @probes.setter
    def probes(self, value):
        t = _native.torch()
        # numpy arrays (the reference's type, engine.py:219-223) or tensors
        stack = t.stack([(v if isinstance(v, t.Tensor) else t.as_tensor(np.asarray(v)))
                         .to(self.obj.device, self.obj.dtype) for v in value])
        if self.frame_chirp is not None:
            stack = stack * self.frame_chirp
        self.probe_stack = stack.contiguous()

    @property
    def iteration(self) -> int:
        return len(self.error_trace)

    @property
    def window(self) -> int:
        return int(self.probe_stack.shape[-1])

    def buffer(self, name, shape, dtype, pinned: bool = False):
        """Per-state scratch reused across sweeps: device buffers (visit order,
        status, error terms, posref staging) or pinned host mirrors."""
        t = _native.torch()
        key = (name, pinned)
        b = self._buf.get(key)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            if pinned:
                b = t.empty(shape, dtype=dtype, pin_memory=True)
            else:
                b = t.empty(shape, dtype=dtype, device=self.obj.device)
            self._buf[key] = b
        return b

    def to_numpy(self) -> dict:
        """Host copy in the reference's types (complex128 / float64 numpy)."""
        out = {"obj": self.obj.cpu().numpy().astype(np.complex128),
               "probes": [p.cpu().numpy().astype(np.complex128) for p in self.probes],
               "positions": self.positions.cpu().numpy(),
               "canvas_origin": self.canvas_origin,
               "error_trace": list(self.error_trace)}
        if self.adam is not None:
            out["adam_m"], out["adam_v"], out["adam_t"] = self.adam.numpy()
        return out


def _anchor(position_xy) -> tuple[int, int]:
    """engine.py:69-70 (Python round: half to even)."""
    return int(round(float(position_xy[1]))), int(round(float(position_xy[0])))


def _dtypes(precision: str):
    t = _native.torch()
    return (t.complex64, t.float32) if precision == "fp32" else (t.complex128, t.float64)


_SHADOWS: dict = {}


def _shadow(dataset):
    """Our PtychoDataset for a foreign dataset object (e.g. ptychokit's): it
    carries the cached device copies; dropped when the original dies."""
    from .dataio import PtychoDataset
    if isinstance(dataset, PtychoDataset):
        return dataset
    key = id(dataset)
    ent = _SHADOWS.get(key)
    if ent is None or ent[0]() is not dataset or ent[1].patterns is not dataset.patterns:
        shadow = PtychoDataset(dataset.patterns, dataset.positions, dataset.geometry)
        try:
            ref = weakref.ref(dataset, lambda _r, k=key: _SHADOWS.pop(k, None))
        except TypeError:
            ref = (lambda d=dataset: d)
        _SHADOWS[key] = (ref, shadow)
        ent = _SHADOWS[key]
    return ent[1]


def device_patterns(dataset, real_dtype):
    """The dataset's diffraction stack in HBM (uploaded once, I >= 0 checked)."""
    return _shadow(dataset).device_patterns(real_dtype)


def device_patterns_t(dataset, real_dtype):
    """Per-pattern transposed copy I^T[j][kc][u] (the column passes' layout)."""
    return _shadow(dataset).device_patterns_t(real_dtype)


def initialize(dataset, config: SolverConfig) -> ReconState:
    """engine.py:73-101 -- unit object on the anchor bounding box, mode 1 =
    back-propagated mean amplitude, extra modes = 1%-power orthogonalised
    perturbations (float64 on the GPU, then rounded to the working precision)."""
    t = _native.torch()
    dev = _native.device()
    w = dataset.geometry.window
    check_window(w)
    cdt, rdt = _dtypes(config.precision)
    anchors = np.stack([_anchor(p) for p in dataset.positions])
    origin = anchors.min(axis=0)
    extent = anchors.max(axis=0) - origin + w
    obj = t.ones((int(extent[0]), int(extent[1])), dtype=cdt, device=dev)
    pats = device_patterns(dataset, rdt)
    m = config.mode_count
    noise = None
    if m > 1:
        host = np.empty((m - 1, w, w), dtype=np.complex128)
        for p in range(1, m):
            rng = np.random.default_rng([config.init_seed, p])
            host[p - 1] = rng.standard_normal((w, w)) + 1j * rng.standard_normal((w, w))
        noise = t.from_numpy(host).to(dev)
    probes = t.empty((m, w, w), dtype=cdt, device=dev)
    _native.init_probes(probes, pats, noise, w, m)
    positions = t.from_numpy(np.asarray(dataset.positions, dtype=np.float64).copy()).to(dev)
    adam = AdamBuffers.zeros(dataset.n_positions, dev) if config.posref is not None else None
    # Fresnel: the back-propagated mean amplitude is conj(Q) * P^-1(sqrt(mean I)),
    # i.e. exactly the far-field initial probe in the kernels' P*Q frame (the
    # mode Gram-Schmidt is invariant under the common unit-modulus factor)
    chirp = None
    if config.propagator == "fresnel":
        from .fields import fresnel_chirp
        chirp = fresnel_chirp(dataset.geometry, cdt, dev)
    return ReconState(obj=obj, probes=probes, positions=positions,
                      canvas_origin=(int(origin[0]), int(origin[1])), adam=adam, frame_chirp=chirp)


# ------------------------------------------------ per-visit public functions --
# The reference's visit building blocks (engine.py:104-150), one CUDA call each
# (pty_magnitude_correct / pty_update_object / pty_update_probe).  numpy inputs
# run in complex128 and return numpy (the reference's types); torch inputs keep
# their precision and device and return tensors.  sweep() does not use them: it
# evaluates the same expressions fused in one launch.

def _is_tensor(a) -> bool:
    return isinstance(a, _native.torch().Tensor)


def _visit_dtype(*arrays):
    t = _native.torch()
    for a in arrays:
        if _is_tensor(a) and a.dtype in (t.complex64, t.float32):
            return t.complex64, t.float32
    return t.complex128, t.float64


def _stack(fields, cdt):
    t = _native.torch()
    if _is_tensor(fields):
        x = fields
    else:
        x = t.stack([f if _is_tensor(f) else t.from_numpy(np.asarray(f, np.complex128)) for f in fields])
    return x.to(_native.device(), cdt).contiguous()


def _field(a, dt):
    t = _native.torch()
    x = a if _is_tensor(a) else t.from_numpy(np.ascontiguousarray(np.asarray(a)))
    return x.to(_native.device(), dt).contiguous()


def _check_visit(w, *shapes):
    from .fields import check_window
    check_window(w)
    for sh in shapes:
        if tuple(sh[-2:]) != (w, w):
            raise ShapeError(f"visit fields must all be {w}x{w}, got {tuple(sh)}")


def magnitude_correct(probes, o_j, i_j, epsilon_rel: float = 1e-12):
    """engine.py:104-120 -- mixed-state modulus constraint on the GPU.

    Returns (corrected exit waves, original detector waves) as lists of M
    fields; raises DataError for negative intensities (engine.py:111-112)."""
    t = _native.torch()
    cdt, rdt = _visit_dtype(o_j, probes if _is_tensor(probes) else (probes[0] if len(probes) else None))
    p = _stack(probes, cdt)
    o = _field(o_j, cdt)
    i = _field(i_j, rdt)
    w = o.shape[-1]
    _check_visit(w, p.shape, o.shape, i.shape)
    corrected = t.empty_like(p)
    psi = t.empty_like(p)
    status = t.zeros(1, dtype=t.int32, device=o.device)
    _native.magnitude_correct(p, o, i, epsilon_rel, corrected, psi, status)
    raise_for_status(int(status.item()), "magnitude_correct")
    if _is_tensor(o_j):
        return list(corrected.unbind(0)), list(psi.unbind(0))
    c, d = corrected.cpu().numpy(), psi.cpu().numpy()
    return [c[k] for k in range(c.shape[0])], [d[k] for k in range(d.shape[0])]


def update_object(o_j, probes, psi_corrected, alpha_obj: float, gamma: float,
                  epsilon_rel: float = 1e-12):
    """engine.py:123-137 -- rPIE object update of one crop (gamma = 1: ePIE)."""
    t = _native.torch()
    cdt, _ = _visit_dtype(o_j, probes if _is_tensor(probes) else (probes[0] if len(probes) else None))
    o = _field(o_j, cdt)
    p = _stack(probes, cdt)
    c = _stack(psi_corrected, cdt)
    _check_visit(o.shape[-1], o.shape, p.shape, c.shape)
    out = t.empty_like(o)
    status = t.zeros(1, dtype=t.int32, device=o.device)
    _native.update_object(o, p, c, alpha_obj, gamma, epsilon_rel, out, status)
    raise_for_status(int(status.item()), "update_object")
    return out if _is_tensor(o_j) else out.cpu().numpy()


def update_probe(probe, o_j, psi_corrected, alpha_probe: float, beta: float,
                 epsilon_rel: float = 1e-12):
    """engine.py:140-150 -- rPIE probe update of one mode (beta = 1: ePIE)."""
    t = _native.torch()
    cdt, _ = _visit_dtype(o_j, probe)
    p = _field(probe, cdt)
    o = _field(o_j, cdt)
    c = _field(psi_corrected, cdt)
    _check_visit(o.shape[-1], o.shape, p.shape, c.shape)
    out = t.empty_like(p)
    status = t.zeros(1, dtype=t.int32, device=o.device)
    _native.update_probe(p, o, c, alpha_probe, beta, epsilon_rel, out, status)
    raise_for_status(int(status.item()), "update_probe")
    return out if _is_tensor(probe) else out.cpu().numpy()


_ORDER_CACHE: dict = {}


def visit_order(n: int, config: SolverConfig, iteration: int) -> np.ndarray:
    """engine.py:177-181.  Shuffled orders are memoised (read-only arrays):
    a replica sweep computes the next iteration's orders while its kernel
    runs, so the host work between two sweeps does not include them."""
    if config.position_order == "shuffled":
        key = (int(n), config.shuffle_seed, int(iteration))
        perm = _ORDER_CACHE.get(key)
        if perm is None:
            perm = np.random.default_rng([config.shuffle_seed, iteration]).permutation(n)
            perm.flags.writeable = False
            if len(_ORDER_CACHE) >= 4096:
                _ORDER_CACHE.clear()
            _ORDER_CACHE[key] = perm
        return perm
    return np.arange(n)


def position_bounds(state: ReconState, window: int):
    """engine.py:167-170 -> (xmin, ymin, xmax, ymax)."""
    h, w = state.obj.shape
    r0, c0 = state.canvas_origin
    return float(c0), float(r0), float(c0 + w - window), float(r0 + h - window)


def _engaged(state: ReconState, config: SolverConfig) -> bool:
    return config.posref is not None and state.iteration >= config.posref.warmup_iterations


def sweep(state: ReconState, dataset, config: SolverConfig, group=None) -> ReconState:
    """engine.py:173-243 -- one pass over all positions, mutating ``state``.

    ``config.batch_size > 1`` selects the batched semi-parallel extension
    (oracle/batched.py); ``group`` (a torch.distributed process group) then
    splits every batch across its ranks and all-reduces the update terms."""
    if config.batch_size > 1:
        return sweep_batched(state, dataset, config, group)
    sweep_replicas([state], [dataset], config)
    return state


from .partition import batch_slice, halo_transfers, ownership, rank_shares, row_bands  # noqa: E402


def _exchange_object_terms(obj_acc, owns, xfers, rank, world, group) -> None:
    """Complete a batch's object accumulator on every rank (partition.py):
    halo rows go to their owner (point-to-point), the owner adds them in rank
    order, then every rank's owned rows are all-gathered.  The rows no rank
    touched are zero everywhere already."""
    import torch.distributed as dist
    t = _native.torch()
    host = dist.get_backend(group) == "gloo"          # gloo point-to-point needs host tensors
    flat = obj_acc.view(obj_acc.shape[0], -1)          # [rows][3 * Wc]: a row band is contiguous
    dev = flat.device
    ops, recvs = [], []
    for src, dst, a, b in xfers:
        if src == rank:
            buf = flat[a:b].contiguous()
            ops.append(dist.P2POp(dist.isend, buf.cpu() if host else buf, dst, group))
        elif dst == rank:
            buf = t.empty((b - a, flat.shape[1]), dtype=flat.dtype, device="cpu" if host else dev)
            ops.append(dist.P2POp(dist.irecv, buf, src, group))
            recvs.append((a, b, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for a, b, buf in recvs:                            # xfers order = source rank order
        _native.accumulate(flat[a:b], buf.to(dev).contiguous())
    rows = [hi - lo for lo, hi in owns]
    R = max(rows)
    if R == 0:
        return
    lo, hi = owns[rank]
    send = t.zeros((R, flat.shape[1]), dtype=flat.dtype, device=dev)
    if hi > lo:
        send[:hi - lo].copy_(flat[lo:hi])
    if host:
        send = send.cpu()
    parts = [t.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    for q, (qlo, qhi) in enumerate(owns):
        if q != rank and qhi > qlo:
            flat[qlo:qhi].copy_(parts[q][:qhi - qlo].to(dev))


def sweep_batched(state: ReconState, dataset, config: SolverConfig, group=None) -> ReconState:
    """Batched rPIE sweep (extension; b = config.batch_size).  Every batch is a
    contiguous slice of the visit order; its positions see the batch-start
    state; numerators/denominators are summed and applied once
    (pty_batch_contrib / pty_batch_apply).

    With a process group (``group``, NCCL on GPUs) every batch is split
    spatially across the ranks (partition.py): each rank accumulates the
    update terms of its row band, halo rows are sent to their owners, the
    owned rows are all-gathered and every rank applies the identical update;
    the probe terms are all-reduced.  Error terms are reduced to three
    scalars per rank and summed once per sweep."""
    t = _native.torch()
    t0 = time.perf_counter()
    st, ds = state, dataset
    w, m = st.window, int(st.probe_stack.shape[0])
    n = ds.n_positions
    cdt = st.obj.dtype
    rdt = t.float32 if cdt == t.complex64 else t.float64
    dcode = _native.dtype_code(cdt)
    world, rank = 1, 0
    if group is not None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    engaged = _engaged(st, config)
    sense = _native.SENSE_NONE
    if engaged:
        sense = _native.SENSE_XCORR_A if config.posref.sensor == "XCORR_A" else _native.SENSE_XCORR_B
    pats = device_patterns(ds, rdt)
    pats_t = device_patterns_t(ds, rdt)
    order = visit_order(n, config, st.iteration)
    b = min(config.batch_size, n)
    h, wc = st.obj.shape
    st.obj = st.obj.contiguous()
    st.probe_stack = st.probe_stack.contiguous()
    status = st.buffer("status", (1,), t.int32)
    status.zero_()
    err = st.buffer("err", (3,), t.float64)
    err_part = st.buffer("err_part", (n, w, 3), t.float64)
    err_part.zero_()
    obj_acc = st.buffer("obj_acc", (h, 3, wc), rdt)
    probe_acc = st.buffer("probe_acc", (2 * m + 1, w, w), rdt)
    stage = st.buffer("stage", (n, 2, w, w), cdt) if engaged else None
    ws = _native.workspace(_native.batch_workspace_bytes(dcode, w, m, b, h, wc), "batch")
    upd_probe = int(bool(config.update_probe_modes) and config.alpha_probe > 0)
    # every batch's position list for this rank: the whole batch in visit
    # order (one rank) or this rank's spatial share (partition.py)
    plan, lists = [], []
    if world > 1:
        # anchor rows are fixed for the sweep (engine.py:193, 226-233): one
        # small device-to-host read of the positions per sweep
        rows_h = np.rint(st.positions[:, 1].cpu().numpy()).astype(np.int64) - st.canvas_origin[0]
    off = 0
    for s in range(0, n, b):
        ids = order[s:s + b]
        if world == 1:
            mine, first, owns, xf = ids, 0, None, None
        else:
            rows = rows_h[ids]
            shares = rank_shares(rows, world)
            bands = row_bands(rows, shares, w, h)
            owns = ownership(bands)
            xf = halo_transfers(bands, owns)
            mine = ids[shares[rank]]
            first = sum(len(shares[q]) for q in range(rank))   # distinct err_part rows per rank
        plan.append((off, len(mine), s + first, owns, xf))
        lists.append(np.asarray(mine, np.int32))
        off += len(mine)
    mine_all = np.concatenate(lists) if lists else np.zeros(0, np.int32)
    lst_h = st.buffer("batch_list", (max(1, n),), t.int32, pinned=True)
    lst_h.numpy()[:len(mine_all)] = mine_all
    lst_d = st.buffer("batch_list", (max(1, n),), t.int32)
    lst_d.copy_(lst_h, non_blocking=True)

    def args_for(k0, count, visit0, sense_k):
        return _native.PtyBatchArgs(
            dcode, w, m, n, _native.ptr(st.obj), h, wc, st.canvas_origin[0], st.canvas_origin[1],
            _native.ptr(st.probe_stack), _native.ptr(pats), _native.ptr(pats_t), _native.ptr(st.positions),
            _native.ptr(lst_d) + 4 * k0, count, visit0,
            float(config.alpha_obj), float(config.alpha_probe), float(config.beta),
            float(config.gamma), float(config.epsilon_rel), upd_probe,
            int(bool(config.track_modulus_error)), sense_k, _native.ptr(stage),
            _native.ptr(obj_acc), _native.ptr(probe_acc), _native.ptr(err_part),
            _native.ptr(status), _native.ptr(ws), ws.numel())

    for k0, count, visit0, owns, xf in plan:
        if count > 0:
            _native.batch_contrib(args_for(k0, count, visit0, sense))
        else:
            obj_acc.zero_()
            probe_acc.zero_()
        if world > 1:
            import torch.distributed as dist
            _exchange_object_terms(obj_acc, owns, xf, rank, world, group)
            dist.all_reduce(probe_acc, group=group)
        # every rank applies the same (complete) terms; the XCORR_A staging is
        # only written for this rank's own positions
        _native.batch_apply(args_for(k0 if count > 0 else 0, max(count, 1), min(visit0, n - 1),
                                     sense if count > 0 else _native.SENSE_NONE))
    _native.batch_finalize(err_part, n, w, err)        # this rank's visits (the other rows are zero)
    if world > 1:
        import torch.distributed as dist
        sums = err[:2].clone()
        dist.all_reduce(sums, group=group)
        worst = err[2:].clone()
        dist.all_reduce(worst, op=dist.ReduceOp.MAX, group=group)
        err[:2].copy_(sums)
        err[2:].copy_(worst)
        # per-bit MAX (a MAX of the bitmasks would drop bits: 1 | 4 -> 4)
        bits = ((status >> t.arange(10, device=status.device, dtype=t.int32)) & 1).to(t.int32)
        dist.all_reduce(bits, op=dist.ReduceOp.MAX, group=group)
        status.copy_((bits << t.arange(10, device=status.device, dtype=t.int32)).sum().view(1))
    if engaged and world == 1:
        _refine_positions(st, config.posref, n, w)
    elif engaged:
        # every rank staged (o_j, o'_j) for its own share of each batch; it
        # senses and Adam-steps exactly those positions, then the disjoint
        # updates are merged with ONE masked-sum all-reduce of (positions, m,
        # v, t) (x + 0 is exact) so every rank holds the same state
        _refine_positions(st, config.posref, n, w, index=mine_all)
        import torch.distributed as dist
        ad = st.adam
        mask = t.zeros((n, 1), dtype=t.float64, device=st.positions.device)
        mask[t.from_numpy(mine_all.astype(np.int64)).to(mask.device)] = 1.0
        packed = t.cat([st.positions, ad.m, ad.v, ad.t.to(t.float64).view(-1, 1)], dim=1) * mask
        dist.all_reduce(packed, group=group)
        st.positions.copy_(packed[:, 0:2])
        ad.m.copy_(packed[:, 2:4])
        ad.v.copy_(packed[:, 4:6])
        ad.t.copy_(packed[:, 6].round().to(t.int64))
    if (config.ortho_interval > 0 and m > 1 and (st.iteration + 1) % config.ortho_interval == 0):
        _native.orthogonalize(st.probe_stack)
    he = st.buffer("err", (3,), t.float64, pinned=True)
    hs = st.buffer("status", (1,), t.int32, pinned=True)
    he.copy_(err, non_blocking=True)
    hs.copy_(status, non_blocking=True)
    t.cuda.current_stream().synchronize()
    raise_for_status(int(hs.numpy()[0]), "batched sweep")
    num, den, worst = he.numpy()
    st.error_trace.append(float(num) / max(float(den), TINY))
    if config.track_modulus_error:
        st.modulus_error_trace.append(float(worst))
    st.seconds_per_iteration.append(time.perf_counter() - t0)
    return st


_REPLICA_BUFS: dict = {}


def _replica_buffers(r: int, n: int) -> dict:
    """Per (device, stream, R, N) pinned + device buffers of sweep_replicas."""
    t = _native.torch()
    dev = _native.device()
    key = (dev.index, t.cuda.current_stream(dev).cuda_stream, r, n)
    b = _REPLICA_BUFS.get(key)
    if b is None:
        b = {"order_h": t.empty((r, n), dtype=t.int32, pin_memory=True),
             "order_d": t.empty((r, n), dtype=t.int32, device=dev),
             "status_d": t.empty((r,), dtype=t.int32, device=dev),
             "status_h": t.empty((r,), dtype=t.int32, pin_memory=True),
             "err_d": t.empty((r, 3), dtype=t.float64, device=dev),
             "err_h": t.empty((r, 3), dtype=t.float64, pin_memory=True)}
        _REPLICA_BUFS[key] = b
    return b


def sweep_replicas(states, datasets, config: SolverConfig, orders=None, kernel_events=None):
    """Advance K independent reconstructions by one sweep each in ONE launch.

    Every replica keeps the reference's exact sequential semantics; the K
    visit chains are simply interleaved step by step across the GPU
    (replica mode).  All replicas share window, mode count,
    position count and precision.  ``config`` is one SolverConfig for all
    replicas or one per replica; per-replica configs may differ only in what
    the host decides (shuffle_seed, position_order, init_seed, iterations),
    the update rule itself is shared by the launch."""
    t = _native.torch()
    states = list(states)
    datasets = list(datasets)
    if len(states) != len(datasets) or not states:
        raise ParameterError("need one dataset per state")
    configs = None
    if isinstance(config, (list, tuple)):
        configs = list(config)
        if len(configs) != len(states):
            raise ParameterError("need one config per state")
        shared = ("alpha_obj", "alpha_probe", "beta", "gamma", "epsilon_rel", "update_probe_modes",
                  "track_modulus_error", "posref", "ortho_interval", "precision", "mode_count",
                  "batch_size", "propagator", "subpixel_gather")
        for c in configs[1:]:
            if any(getattr(c, k) != getattr(configs[0], k) for k in shared):
                raise ParameterError("replicas in one launch must share the update rule "
                                     f"({', '.join(shared)})")
        if orders is None:
            orders = [visit_order(d.n_positions, c, st.iteration)
                      for st, d, c in zip(states, datasets, configs)]
        config = configs[0]
    if len(states) > _native.MAX_SLOTS:
        # more replicas than one launch carries: consecutive launches of at
        # most MAX_SLOTS (each replica's sweep is still one launch)
        for lo in range(0, len(states), _native.MAX_SLOTS):
            hi = lo + _native.MAX_SLOTS
            sweep_replicas(states[lo:hi], datasets[lo:hi], config,
                           None if orders is None else orders[lo:hi], kernel_events)
        return states
    t0 = time.perf_counter()
    s0 = states[0]
    w, m = s0.window, int(s0.probe_stack.shape[0])
    n = datasets[0].n_positions
    cdt = s0.obj.dtype
    rdt = t.float32 if cdt == t.complex64 else t.float64
    dcode = _native.dtype_code(cdt)
    engaged = [_engaged(s, config) for s in states]
    sense = _native.SENSE_NONE
    if any(engaged):
        sense = _native.SENSE_XCORR_A if config.posref.sensor == "XCORR_A" else _native.SENSE_XCORR_B
    slots = (_native.PtySlot * len(states))()
    keep = []
    R = len(states)
    # one pinned/device buffer set for the whole replica set: a single H2D
    # of every visit order, one memset of the status words, one D2H of every
    # error triple and status after the launch (instead of 4 tiny copies or
    # kernels per replica on the host's critical path)
    rb = _replica_buffers(R, n)
    perms = {}
    for k, (st, ds) in enumerate(zip(states, datasets)):
        if ds.geometry.window != w or ds.n_positions != n or st.window != w or st.obj.dtype != cdt \
                or st.probe_stack.shape[0] != m:
            raise ShapeError("replicas must share window, mode count, positions and precision")
        if orders is not None:
            rb["order_h"].numpy()[k] = orders[k]
        else:                                  # one permutation per distinct iteration count
            it = st.iteration
            if it not in perms:
                perms[it] = visit_order(n, config, it)
            rb["order_h"].numpy()[k] = perms[it]
    # throughput sweeps (line-task kernel, > 4 replicas) read the visit orders
    # straight from the pinned host buffer (unified addressing; phase 0 turns
    # them into the device step table): no host-to-device copy on the stream,
    # so a sweep never queues behind a bulk upload occupying the copy engine
    # (e.g. the next step's diffraction data).  The latency kernel (<= 4
    # replicas) reads the order every step and gets a device copy.
    host_order = R > 4 and not config.subpixel_gather
    if not host_order:
        rb["order_d"].copy_(rb["order_h"], non_blocking=True)
    rb["status_d"].zero_()
    for k, (st, ds) in enumerate(zip(states, datasets)):
        pats = device_patterns(ds, rdt)
        pats_t = device_patterns_t(ds, rdt)
        order_d = rb["order_h"][k] if host_order else rb["order_d"][k]
        status = rb["status_d"][k:k + 1]
        err = rb["err_d"][k]
        stage = st.buffer("stage", (n, 2, w, w), cdt) if sense != _native.SENSE_NONE else None
        st.obj = st.obj.contiguous()
        st.probe_stack = st.probe_stack.contiguous()
        h, wc = st.obj.shape
        slots[k] = _native.PtySlot(_native.ptr(st.obj), h, wc, st.canvas_origin[0], st.canvas_origin[1],
                                   _native.ptr(st.probe_stack), _native.ptr(pats), _native.ptr(pats_t),
                                   _native.ptr(st.positions), _native.ptr(order_d),
                                   _native.ptr(stage), _native.ptr(err), _native.ptr(status))
        keep.append((pats, pats_t, order_d))
    nbytes = _native.sweep_workspace_bytes(dcode, w, m, n, len(states))
    ws = _native.workspace(nbytes)
    args = _native.PtySweepArgs(
        dcode, w, m, n, len(states), slots,
        float(config.alpha_obj), float(config.alpha_probe), float(config.beta), float(config.gamma),
        float(config.epsilon_rel), int(bool(config.update_probe_modes) and config.alpha_probe > 0),
        int(bool(config.track_modulus_error)), sense, _native.ptr(ws), ws.numel())
    if kernel_events is not None:
        kernel_events[0].record()
    if config.subpixel_gather:
        _native.sweep_subpixel(args)
    else:
        _native.sweep(args)
    if kernel_events is not None:
        kernel_events[1].record()

    for st, eng in zip(states, engaged):
        if eng:
            _refine_positions(st, config.posref, n, w)
    for st in states:
        if (config.ortho_interval > 0 and st.probe_stack.shape[0] > 1
                and (st.iteration + 1) % config.ortho_interval == 0):
            _native.orthogonalize(st.probe_stack)
    # the next sweep's visit orders, computed while this one runs on the GPU
    for st, c in zip(states, configs if configs is not None else [config] * len(states)):
        visit_order(n, c, st.iteration + 1)

    rb["err_h"].copy_(rb["err_d"], non_blocking=True)
    rb["status_h"].copy_(rb["status_d"], non_blocking=True)
    t.cuda.current_stream().synchronize()
    dt = time.perf_counter() - t0
    err_h, status_h = rb["err_h"].numpy(), rb["status_h"].numpy()
    for k, st in enumerate(states):
        (num, den, worst), status = err_h[k], status_h[k]
        raise_for_status(int(status), f"sweep, replica {k}")
        st.error_trace.append(float(num) / max(float(den), TINY))
        if config.track_modulus_error:
            st.modulus_error_trace.append(float(worst))
        st.seconds_per_iteration.append(dt)
    return states


def _refine_positions(st: ReconState, pc: PosRefConfig, n: int, w: int, index=None) -> None:
    """posref.py:57-113 for every position of the sweep, batched: register the
    staged pairs (XCORR_A: o_j vs o'_j; XCORR_B: modelled vs measured
    intensity) with raw weighting, then the float64 Adam step + clamp.
    ``index`` (int32 numpy, optional): only these positions were staged."""
    t = _native.torch()
    stage = st.buffer("stage", (n, 2, w, w), st.obj.dtype)
    idx_d = None
    if index is not None:
        idx_d = t.from_numpy(np.ascontiguousarray(index, np.int32)).to(stage.device)
        stage = stage.index_select(0, idx_d.long())
        n = int(idx_d.numel())
    dy = st.buffer("reg_dy", (n,), t.float64)
    dx = st.buffer("reg_dx", (n,), t.float64)
    peak = st.buffer("reg_peak", (n,), t.float64)
    ok = st.buffer("reg_ok", (n,), t.int32)
    if stage.dtype == t.complex128:
        _native.register_batch(stage, w, n, 1, int(pc.kappa), dy, dx, peak, ok)
    else:
        # register in float64 like the reference (its crops are complex128,
        # registration.py:123-128): fp32 correlation peaks of near-identical
        # crops are too flat to resolve the 1/kappa grid; the complex64 pairs
        # are widened while the first kernel loads them (no conversion pass)
        chunk = max(1, min(n, (1 << 30) // (2 * w * w * 16)))
        work = st.buffer("stage64", (chunk, 2, w, w), t.complex128)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            _native.register_batch(work[:e - s], w, e - s, 1, int(pc.kappa),
                                   dy[s:e], dx[s:e], peak[s:e], ok[s:e], pairs_c64=stage[s:e])
    # sensors return (gx, gy) = (est.dx, est.dy) (posref.py:63)
    _native.adam_apply(st.positions, st.adam, dx, dy, ok, pc, position_bounds(st, w), index=idx_d)


def resume(checkpoint_dir, dataset, config: SolverConfig) -> ReconState:
    """Rebuild a device-resident ReconState from a checkpoint written by
    ``run(checkpoint_every=...)`` (dataio.py:164-204 format, plus the Adam
    buffers this package stores), so a reconstruction continues where it
    stopped: same visit order (iteration = len(error_trace)), positions and
    Adam state.  The container stores complex64 fields (as the reference)."""
    t = _native.torch()
    ck = read_checkpoint(checkpoint_dir)
    dev = _native.device()
    cdt = t.complex128 if config.precision == "fp64" else t.complex64
    w = dataset.geometry.window
    chirp = None
    if config.propagator == "fresnel":
        from .fields import fresnel_chirp
        chirp = fresnel_chirp(dataset.geometry, cdt, dev)
    obj = t.from_numpy(np.ascontiguousarray(ck["object"])).to(dev, cdt)
    positions = t.from_numpy(np.ascontiguousarray(ck["positions"], np.float64)).to(dev)
    if positions.shape != (dataset.n_positions, 2):
        raise ShapeError(f"checkpoint has {positions.shape[0]} positions, dataset {dataset.n_positions}")
    adam = None
    if config.posref is not None:
        if "adam" in ck:
            m, v, tt = ck["adam"]
            adam = AdamBuffers(t.from_numpy(np.ascontiguousarray(m)).to(dev),
                               t.from_numpy(np.ascontiguousarray(v)).to(dev),
                               t.from_numpy(np.ascontiguousarray(tt, np.int64)).to(dev))
        else:
            adam = AdamBuffers.zeros(dataset.n_positions, dev)
    st = ReconState(obj=obj, probes=t.zeros((len(ck["probes"]), w, w), dtype=cdt, device=dev),
                    positions=positions, canvas_origin=ck["canvas_origin"], adam=adam,
                    error_trace=ck["error_trace"], frame_chirp=chirp)
    st.probes = [np.asarray(p) for p in ck["probes"]]
    return st


def run(dataset, config: SolverConfig, state: ReconState | None = None,
        checkpoint_every: int = 0, checkpoint_dir=None) -> ReconState:
    """engine.py:246-260."""
    if state is None:
        state = initialize(dataset, config)
    for _ in range(config.iterations):
        sweep(state, dataset, config)
        if (checkpoint_every > 0 and checkpoint_dir is not None
                and state.iteration % checkpoint_every == 0):
            snap = Path(checkpoint_dir) / f"iter_{state.iteration:04d}"
            write_checkpoint(snap, state.obj, state.probes, state.positions, state.canvas_origin,
                             state.error_trace, state.iteration,
                             adam=None if state.adam is None else (state.adam.m, state.adam.v, state.adam.t))
    return state
