#!/usr/bin/env python
"""rPIE sweep benchmark (BASELINE.json metric: diffraction positions/s per
rPIE iteration at 256x256x3 modes; % HBM roofline).

Workload (BASELINE.json configs[1]): simulated 20x20 scan
(400 positions), 256x256 patterns, 3 mixed-state probe modes, rPIE
(alpha 0.9, beta = gamma = 0.5), far field, shuffled order.  A step is one rPIE
iteration (one sweep over all 400 positions).  Each GPU runs R independent
reconstructions of that dataset in exact reference (sequential) order,
interleaved in one cooperative launch per sweep ("replica mode");
R = 1 is the single-reconstruction latency figure, also reported.  Default
R = 18: the row-update phase has R * W/4 team tasks and the grid has
148 SMs x 2 CTAs x 4 teams = 1184 teams, so 18 x 64 = 1152 is the largest R
that finishes that phase in one round (measured: R = 18 250 K pos/s,
R = 20 173 K pos/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--replicas R]
    python bench.py --impl reference ...   # the reference algorithm on host cores
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (one rank per GPU,
replicas only -- the sequential path does not shard; weak scaling).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

W, M, GRID, STEP_PX, RADIUS = 256, 3, (20, 20), 32.0, 60.0
POWERS = (0.8, 0.1, 0.1)
B_POS = W * W * (20 + 16 * M)        # algorithmic bytes per position
# algorithmic FFT flops per position: 2M 2-D transforms of W x W at 5 N log2 N
# ("algorithmic flops per position"); 31.5 MFLOP at 256^2 x 3
FFT_FLOP_POS = 2 * M * 5 * W * W * int(math.log2(W * W))
METRIC = "diffraction positions/sec per rPIE iteration at 256x256x3 modes; % HBM roofline"
WORKLOAD = ("config 2: simulated 20x20 scan (400 positions), 256x256 patterns, 3 mixed-state "
            "probe modes, rPIE alpha=0.9 beta=gamma=0.5, Fraunhofer, shuffled order")


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def fp32_peak_tflops():
    """FP32 FMA peak, derived (not measured): 148 SMs x 128 lanes x 2 flop x max SM clock."""
    mhz = 1965.0
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        mhz = float(json.loads(p.read_text()).get("sm_max_mhz", mhz))
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def solver_config(precision="fp32"):
    import paper_2205_04295_b200 as pk
    return pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=M,
                           position_order="shuffled", shuffle_seed=0, precision=precision)


def replica_configs(cfg, R, rank):
    """One config per replica: its own init_seed AND shuffle_seed (independent
    reconstructions, each in exact reference order)."""
    import paper_2205_04295_b200 as pk
    return [pk.SolverConfig(**{**cfg.__dict__, "init_seed": rank * 1000 + r, "shuffle_seed": rank * 1000 + r})
            for r in range(R)]


def make_dataset(seed=1):
    import paper_2205_04295_b200 as pk
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, W)
    plan = pk.make_scan(GRID, STEP_PX, 1.0, seed=seed)
    obj = pk.make_object(pk.canvas_shape_for(plan, W), "spokes", seed=seed)
    probes = pk.make_probe(pk.ProbeSpec(M, POWERS, "disk", RADIUS), geom)
    ds = pk.synthesize(obj, probes, plan, geom, noise="none", seed=seed)
    ds.patterns = ds.patterns.astype(np.float32)          # the container's on-disk precision
    return ds


# ------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region.

    nvidia-smi is started before the warm-up (its start-up alone can outlast
    a short timed region); every sample is stamped on arrival and the summary
    keeps the samples between mark_start() and mark_end() (plus one polling
    interval), falling back to the samples nearest the region if none landed
    inside it."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    PERIOD_MS = 50

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def mark_start(self):
        self.t0 = time.monotonic()

    def mark_end(self):
        self.t1 = time.monotonic()
        # make sure at least two samples exist after the region started
        deadline = self.t1 + 2.0
        while self.proc is not None and time.monotonic() < deadline and \
                sum(1 for t, _ in self.lines if t >= self.t0) < 2:
            time.sleep(0.02)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        lines = self.lines
        if self.t0 is not None and self.t1 is not None:
            inside = [(t, ln) for t, ln in lines if self.t0 <= t <= self.t1 + self.PERIOD_MS / 1e3]
            lines = inside or sorted(lines, key=lambda x: min(abs(x[0] - self.t0), abs(x[0] - self.t1)))[:2]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def flush_l2(buf):
    buf.add_(1)      # 256 MiB read+write > 126 MB L2


# ------------------------------------------------------------ GPU arm -----
def run_states(states, datasets, cfgs, kernel_events=None):
    import paper_2205_04295_b200 as pk
    pk.sweep_replicas(states, datasets, cfgs, kernel_events=kernel_events)


def gpu_arm(args, rank, world):
    import torch
    import paper_2205_04295_b200 as pk
    from paper_2205_04295_b200 import _native

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg = solver_config(args.precision)
    R = args.replicas
    # every replica is an independent reconstruction of its OWN dataset (scan
    # jitter, object and synthesised patterns from seed 1 + rank*1000 + r) with
    # its own init and shuffle seeds, so no two replicas share inputs or order
    dsets = [make_dataset(seed=1 + rank * 1000 + r) for r in range(R)]
    cfgs = replica_configs(cfg, R, rank)
    ds = dsets[0]
    n = ds.n_positions
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # ---- value: R replicas resident in HBM, device-timed sweeps
    states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
    with ClockSampler(dev.index) as clocks:
        for _ in range(args.warmup):
            run_states(states, dsets, cfgs)
        torch.cuda.synchronize()
        step_ms, kern_ms = [], []
        launches0 = _native.launch_count()
        clocks.mark_start()
        for _ in range(args.steps):
            flush_l2(flush)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run_states(states, dsets, cfgs, kernel_events=(k0, k1))
            e1.record()
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            kern_ms.append(k0.elapsed_time(k1))
        clocks.mark_end()
    launches = _native.launch_count() - launches0
    total_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([total_ms, sum(kern_ms)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, kern_total = t.tolist()
    else:
        kern_total = sum(kern_ms)
    positions = R * n * args.steps * world
    value = positions / (total_ms / 1e3)
    kernel_s = kern_total / 1e3 / args.steps                 # per sweep launch (R*n positions)
    hbm, peak_kind = peaks()
    achieved = R * n * B_POS / kernel_s / 1e9
    fft_tflops = R * n * FFT_FLOP_POS / kernel_s / 1e12
    traffic = None
    tp = ROOT / "profiles" / "sweep_traffic.json"
    if tp.exists():
        tj = json.loads(tp.read_text())
        if tj.get("replicas") == R and tj.get("window") == W:
            traffic = tj.get("dram_bytes_per_launch")

    # ---- single reconstruction (R = 1): the reference's own sequential case
    single = None
    if R != 1 and not args.no_single:
        st1 = [pk.initialize(ds, cfgs[0])]
        for _ in range(2):
            run_states(st1, [ds], cfgs[:1])
        ms1 = []
        for _ in range(max(3, args.steps // 2)):
            flush_l2(flush)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run_states(st1, [ds], cfgs[:1])
            b.record()
            torch.cuda.synchronize()
            ms1.append(a.elapsed_time(b))
        mean1 = statistics.mean(ms1)
        single = {"positions_per_s": n / (mean1 / 1e3), "iterations_per_s": 1e3 / mean1,
                  "us_per_visit": mean1 * 1e3 / n, "ms_per_iteration": mean1}

    # ---- e2e: the public API on HOST buffers; H2D of the step's inputs and
    # D2H of its result inside the timed region, every step
    e2e = e2e_arm(args, states, dsets, cfgs, dev, world)
    fp64 = None
    if args.precision == "fp32" and not args.no_fp64:
        fp64 = fp64_leg(args, dsets, dev, world, flush)
    return dict(fp64=fp64, value=value, ms_per_step=total_ms / args.steps, kernel_ms=kern_total / args.steps,
                achieved=achieved, fft_tflops=fft_tflops, hbm=hbm, peak_kind=peak_kind, traffic=traffic, clocks=clocks.summary(),
                launches=launches, single=single, e2e=e2e, n=n)


def fp64_leg(args, dsets, dev, world, flush):
    """The same workload (same R distinct datasets and seeds) through the
    complex128 instantiation of the sweep kernel -- the reference's own
    precision, beside the fp64 reference arm."""
    import torch
    import paper_2205_04295_b200 as pk
    R = len(dsets)
    cfgs = replica_configs(solver_config("fp64"), R, int(os.environ.get("RANK", 0)))
    states = [pk.initialize(d, c) for d, c in zip(dsets, cfgs)]
    for _ in range(2):
        run_states(states, dsets, cfgs)
    ms = []
    for _ in range(max(2, args.steps // 3)):
        flush_l2(flush)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run_states(states, dsets, cfgs)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    total = sum(ms)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total = t.item()
    per = total / len(ms)
    n = dsets[0].n_positions
    hbm, _ = peaks()
    v = R * n * world / (per / 1e3)
    del states
    torch.cuda.empty_cache()
    return {"dtype": "c128", "replicas": R, "value": v, "unit": "positions/s", "ms_per_step": per,
            "roofline_frac_c64_bytes": v * B_POS / (hbm * 1e9 * world),
            "note": "complex128 kernels (2x the bytes of the c64 B_pos the roofline uses)"}


def e2e_arm(args, states, dsets, cfgs, dev, world):
    """The public API fed from HOST memory every step: every replica's input
    (its own diffraction stack, pinned host float32) is copied to the device
    and re-laid out (the transposed copy the column passes stream), the R
    reconstructions sweep, and the step's result (every replica's error
    metric and status word) is read back -- all inside the timed region, which
    spans the K steps as one region (the first step's copy is not overlapped).
    The reconstruction state stays resident on the device between steps, as a
    user's does."""
    import torch
    import paper_2205_04295_b200 as pk
    R = len(states)
    hosts = [torch.from_numpy(np.ascontiguousarray(d.patterns, np.float32)).pin_memory() for d in dsets]
    dxs = [pk.PtychoDataset(patterns=d.patterns, positions=d.positions, geometry=d.geometry) for d in dsets]
    for x in dxs:                                           # the datasets' device buffers exist (validated once)
        pk.engine.device_patterns_t(x, torch.float32)
    # every step's H2D lands directly in one of two raw device buffer sets (copy
    # stream, copy engines) while the previous step sweeps; the step then lays
    # out its transposed copy (the column passes' layout) and points the
    # datasets at its buffers -- no device-to-device staging copy
    main = torch.cuda.current_stream()
    cstream = torch.cuda.Stream()
    raw = [[torch.empty(h.shape, dtype=torch.float32, device=dev) for h in hosts] for _ in range(2)]
    pt = [torch.empty(h.shape, dtype=torch.float32, device=dev) for h in hosts]
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    used = [False, False]
    key = str(torch.float32)

    def issue_copy(i):
        slot = i % 2
        if used[slot]:
            cstream.wait_event(consumed[slot])
        with torch.cuda.stream(cstream):
            for d_, h in zip(raw[slot], hosts):
                d_.copy_(h, non_blocking=True)                       # H2D: step i's inputs
            copied[slot].record(cstream)

    def run_steps(n):
        issue_copy(0)
        for i in range(n):
            slot = i % 2
            main.wait_event(copied[slot])
            if i + 1 < n:
                issue_copy(i + 1)
            for r, x in enumerate(dxs):
                pt[r].copy_(raw[slot][r].transpose(1, 2))             # device re-layout
                x._device[(key, id(x.patterns))] = raw[slot][r]
                x._device[("T", key, id(x.patterns))] = pt[r]
            consumed[slot].record(main)
            used[slot] = True
            pk.sweep_replicas(states, dxs, cfgs)                     # ends with the D2H of the metric

    run_steps(args.warmup)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run_steps(args.steps)
    b.record()
    torch.cuda.synchronize()
    total = a.elapsed_time(b)
    h2d = sum(h.numel() * 4 for h in hosts)
    d2h = R * (3 * 8 + 4)                                          # error triple + status per replica
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total = t.item()
    value = R * dsets[0].n_positions * args.steps * world / (total / 1e3)
    return {"value": value, "unit": "positions/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": total / args.steps,
            "inputs": f"{R} distinct diffraction stacks uploaded every step"}


# ------------------------------------------- other named configs (1, 3, 4) ----
CONFIGS = {
    # BASELINE.json configs[0], [2], [3]
    "config1": dict(W=128, M=1, grid=(10, 10), step=16.0, radius=30.0, powers=(1.0,), lam=8.3187e-10,
                    posref=False, propagator="farfield"),
    "config3": dict(W=256, M=3, grid=(20, 20), step=32.0, radius=60.0, powers=(0.8, 0.1, 0.1), lam=8.3187e-10,
                    posref=True, propagator="farfield", replicas=18, distinct_data=True),
    "config4": dict(W=512, M=5, grid=(40, 40), step=64.0, radius=120.0, powers=(0.8, 0.05, 0.05, 0.05, 0.05),
                    lam=8.29e-10, posref=True, propagator="fresnel", replicas=9, distinct_data=False),
}


def configs_leg(args):
    """Single-reconstruction throughput (exact reference order) of the other
    named shapes: positions/s, iterations/s and the algorithmic-bytes
    roofline fraction.  Config 3/4: +-2 px injected position errors, posref
    XCORR_A kappa=10 engaged from the first sweep; config 4 with the Fresnel
    propagator (extension)."""
    import torch
    import paper_2205_04295_b200 as pk
    hbm, _ = peaks()
    out = {}
    for name, c in CONFIGS.items():
        try:
            w, m = c["W"], c["M"]
            geom = pk.Geometry.create(c["lam"], 0.75, 20e-6, w)
            plan = pk.make_scan(c["grid"], c["step"], 1.0, seed=1)
            obj = pk.make_object(pk.canvas_shape_for(plan, w), "spokes", seed=1)
            probes = pk.make_probe(pk.ProbeSpec(m, c["powers"], "disk", c["radius"]), geom)
            ds = pk.synthesize(obj, probes, plan, geom, noise="none", seed=1, propagator=c["propagator"])
            ds.patterns = ds.patterns.astype(np.float32)
            if c["posref"]:
                ds.positions = ds.positions + np.random.default_rng(42).uniform(-2, 2, ds.positions.shape)
            posref = pk.PosRefConfig(sensor="XCORR_A", kappa=10, warmup_iterations=0) if c["posref"] else None
            cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=m,
                                  position_order="shuffled", shuffle_seed=0, precision=args.precision,
                                  posref=posref, propagator=c["propagator"])
            st = pk.initialize(ds, cfg)
            for _ in range(2):
                pk.sweep(st, ds, cfg)
            steps = 3 if w >= 512 else 5
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(steps):
                pk.sweep(st, ds, cfg)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e) / steps
            n = ds.n_positions
            bpos = w * w * (20 + 16 * m)
            out[name] = {"window": w, "modes": m, "positions": n, "posref": c["posref"],
                         "propagator": c["propagator"], "positions_per_s": n / (ms / 1e3),
                         "iterations_per_s": 1e3 / ms, "ms_per_iteration": ms,
                         "roofline_frac": n / (ms / 1e3) * bpos / (hbm * 1e9),
                         "error_trace_last": st.error_trace[-1]}
            R = c.get("replicas", 0)
            if R > 1 and not args.no_config_replicas:
                # replica mode: R independent reconstructions in one launch per
                # sweep (own init and shuffle seeds; config 3: own datasets too)
                del st
                torch.cuda.empty_cache()
                if c.get("distinct_data"):
                    dsets = [ds]
                    for r in range(1, R):
                        pl = pk.make_scan(c["grid"], c["step"], 1.0, seed=1 + r)
                        ob = pk.make_object(pk.canvas_shape_for(pl, w), "spokes", seed=1 + r)
                        d = pk.synthesize(ob, probes, pl, geom, noise="none", seed=1 + r,
                                          propagator=c["propagator"])
                        d.patterns = d.patterns.astype(np.float32)
                        if c["posref"]:
                            d.positions = d.positions + np.random.default_rng(42 + r).uniform(-2, 2, d.positions.shape)
                        dsets.append(d)
                    shared = "own dataset, init and shuffle seed per replica"
                else:
                    dsets = [ds] * R
                    shared = "one dataset, own init and shuffle seed per replica"
                cfgs = replica_configs(cfg, R, 0)
                sts = [pk.initialize(d, cc) for d, cc in zip(dsets, cfgs)]
                for _ in range(2):
                    pk.sweep_replicas(sts, dsets, cfgs)
                rsteps = 2 if w >= 512 else 4
                torch.cuda.synchronize()
                a.record()
                for _ in range(rsteps):
                    pk.sweep_replicas(sts, dsets, cfgs)
                e.record()
                torch.cuda.synchronize()
                rms = a.elapsed_time(e) / rsteps
                out[name]["replicas"] = {"replicas": R, "data": shared, "positions_per_s": R * n / (rms / 1e3),
                                         "ms_per_iteration": rms,
                                         "roofline_frac": R * n / (rms / 1e3) * bpos / (hbm * 1e9),
                                         "error_trace_last_max": max(x.error_trace[-1] for x in sts)}
                del sts
        except Exception as exc:                      # report, never lose the main line
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        finally:
            torch.cuda.empty_cache()
    return out


# ----------------------------------------------- batched leg (config 5) ----
def batched_leg(args, rank, world):
    """BASELINE configs[4]: batched semi-parallel rPIE, 6400 positions of
    256x256x3; every batch is split across the ranks and the update terms are
    all-reduced (NCCL) once per batch (strong scaling over ranks)."""
    import torch
    import paper_2205_04295_b200 as pk
    global GRID
    grid0 = GRID
    GRID = (80, 80)
    try:
        ds = make_dataset(seed=5)
    finally:
        GRID = grid0
    n = ds.n_positions
    b = args.batch
    cfg = pk.SolverConfig(**{**solver_config(args.precision).__dict__, "batch_size": b})
    group = torch.distributed.group.WORLD if world > 1 else None
    st = pk.initialize(ds, cfg)
    for _ in range(2):
        pk.sweep(st, ds, cfg, group=group)
    ms = []
    for _ in range(max(2, args.steps // 2)):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pk.sweep(st, ds, cfg, group=group)
        e.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(e))
    total = sum(ms)
    if world > 1:
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total = t.item()
    per = total / len(ms)
    hbm, _ = peaks()
    value = n / (per / 1e3)
    return {"workload": "config 5: batched semi-parallel rPIE, 80x80 scan (6400 positions), 256x256x3 modes, "
                        f"batch {b} split spatially over {world} GPU(s): halo rows to their owner + all-gather of owned rows, probe terms all-reduced (partition.py)",
            "value": value, "unit": "positions/s", "ms_per_iteration": per, "iterations_per_s": 1e3 / per,
            "scaling": "strong", "roofline_frac": value * B_POS / (hbm * 1e9 * world),
            "error_trace_last": st.error_trace[-1]}


# ------------------------------------------------------- CPU reference ----
def _cpu_worker(payload):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as _np
    from oracle import rpie
    patterns, positions, probes, cfg_kw, sample = payload

    class Cfg:
        pass
    cfg = Cfg()
    for k, v in cfg_kw.items():
        setattr(cfg, k, v)
    st = rpie.initialize(patterns, positions, W, cfg)
    st.probes = [_np.asarray(p, _np.complex128) for p in probes]
    t0 = time.perf_counter()
    rpie.sweep(st, patterns, W, cfg, order=_np.arange(sample))
    return sample, time.perf_counter() - t0


def cpu_sample_payload(sample):
    ds = make_dataset_host(sample)
    cfg_kw = dict(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=M,
                  position_order="fixed", shuffle_seed=0, init_seed=0, epsilon_rel=1e-12,
                  ortho_interval=0, update_probe_modes=True, posref=None, track_modulus_error=False)
    return ds, cfg_kw


def make_dataset_host(sample):
    """The first `sample` positions of the config-2 dataset, synthesised on the
    host with numpy (the reference arm never touches the GPU path)."""
    import paper_2205_04295_b200.simulate as sim
    from oracle import rpie
    import paper_2205_04295_b200 as pk
    geom = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, W)
    plan = sim.make_scan(GRID, STEP_PX, 1.0, seed=1)
    obj = sim.make_object(sim.canvas_shape_for(plan, W), "spokes", seed=1)
    probes = sim.make_probe(sim.ProbeSpec(M, POWERS, "disk", RADIUS), geom)
    fy = np.fft.fftfreq(W)[:, None]
    fx = np.fft.fftfreq(W)[None, :]
    pats = np.empty((sample, W, W))
    for j in range(sample):
        x, y = plan.true_positions[j]
        ar, ac = int(round(y)), int(round(x))
        view = obj[ar:ar + W, ac:ac + W]
        view = np.fft.ifft2(np.fft.fft2(view) * np.exp(-2j * np.pi * (fy * -(y - ar) + fx * -(x - ac))))
        pats[j] = sum(np.abs(rpie.centered_fft2(p * view)) ** 2 for p in probes)
    pats = pats.astype(np.float32).astype(np.float64)
    return pats, np.asarray(plan.nominal[:sample], np.float64)


def cpu_reference(workers, sample, repeats):
    """The reference algorithm (oracle port, numpy float64, one process per core)
    on `workers` host cores, each sweeping `sample` positions of config 2."""
    import multiprocessing as mp
    (pats, pos), cfg_kw = cpu_sample_payload(sample)
    # initial probes as the reference would build them (mode noise etc.)
    from oracle import rpie

    class Cfg:
        pass
    cfg = Cfg()
    for k, v in cfg_kw.items():
        setattr(cfg, k, v)
    probes = rpie.initialize(pats, pos, W, cfg).probes
    payload = (pats, pos, probes, cfg_kw, sample)
    ctx = mp.get_context("spawn")
    env_threads = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in env_threads:
        os.environ[k] = "1"
    walls = []
    with ctx.Pool(workers) as pool:
        pool.map(_cpu_worker, [payload] * workers)               # warm the workers
        for _ in range(repeats):
            t0 = time.perf_counter()
            pool.map(_cpu_worker, [payload] * workers)
            walls.append(time.perf_counter() - t0)
    for k, v in env_threads.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    return [workers * sample / w for w in walls]


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ main ----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--replicas", type=int, default=int(os.environ.get("PTY_BENCH_REPLICAS", 18)))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-sample", type=int, default=32)
    ap.add_argument("--cpu-workers", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-single", action="store_true")
    ap.add_argument("--no-batched", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-config-replicas", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--batch", type=int, default=1600)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    cores = host_cores()
    workers = args.cpu_workers or max(1, min(cores, 64))

    if args.impl == "reference":
        if rank != 0:
            return
        vals = cpu_reference(workers, args.cpu_sample, max(1, args.warmup + args.steps))
        vals = vals[args.warmup:] or vals
        v = statistics.mean(vals)
        line = {"metric": METRIC, "value": v, "unit": "positions/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * workers * args.cpu_sample / v,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOAD, "window": W, "modes": M,
                           "positions_per_step": workers * args.cpu_sample,
                           "parallelism": f"{workers} single-thread reference processes"},
                "cpu_baseline": {"value": v, "unit": "positions/s", "cores": workers, "kind": "port",
                                 "sample": f"{args.cpu_sample} positions of config 2 per process, "
                                           f"{workers} processes (oracle/rpie.py numpy float64)"},
                "e2e": {"value": v, "unit": "positions/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        # fixed NCCL algorithm and protocol: the batched mode's collectives then
        # reduce in the same order on every run (bitwise-reproducible sweeps)
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group("nccl")
    res = gpu_arm(args, rank, world)
    batched = None
    if not args.no_batched:
        try:
            batched = batched_leg(args, rank, world)
        except Exception as exc:                      # report, never lose the main line
            batched = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    configs = None
    if rank == 0 and not args.no_configs:
        configs = configs_leg(args)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        vals = cpu_reference(workers, args.cpu_sample, 1)
        cpu = {"value": vals[0], "unit": "positions/s", "cores": workers, "kind": "port",
               "sample": f"{args.cpu_sample} positions of config 2 per process, {workers} "
                         f"single-thread processes on {cores} host cores (oracle/rpie.py, numpy float64)"}
    if rank == 0:
        frac = res["achieved"] / res["hbm"]
        line = {
            "metric": METRIC, "value": res["value"], "unit": "positions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c64" if args.precision == "fp32" else "c128", "data": "synthetic",
            "config": {"workload": WORKLOAD, "window": W, "modes": M, "positions": res["n"],
                       "replicas_per_gpu": args.replicas, "precision": args.precision,
                       "replica_data": "every replica its own dataset (seed 1 + rank*1000 + r), init_seed and shuffle_seed",
                       "parallelism": f"replicas x{args.replicas} per GPU x{world} GPUs",
                       "l2": "256 MiB buffer rewritten between timed steps"},
            "roofline": {"bound": "hbm", "achieved": res["achieved"], "peak": res["hbm"], "unit": "GB/s",
                         "frac": frac, "traffic": res["traffic"],
                         "kernel": "pty::sweep_kernel<float,256> (persistent cooperative sweep)",
                         "bytes_per_position": B_POS, "peak_kind": res["peak_kind"],
                         "kernel_ms_per_step": res["kernel_ms"]},
            "fft": {"bound": "fp32", "achieved": res["fft_tflops"], "peak": fp32_peak_tflops(),
                    "unit": "TFLOP/s", "frac": res["fft_tflops"] / fp32_peak_tflops(),
                    "flops_per_position": FFT_FLOP_POS, "convention": "5 N log2 N per 2-D transform, 2M transforms per visit",
                    "peak_kind": "derived 148 SM x 128 FMA lanes x 2 x sm_max_mhz"},
            "cpu_baseline": cpu,
            "e2e": res["e2e"],
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "single_reconstruction": res["single"],
            "fp64": res["fp64"],
            "batched": batched,
            "configs": configs,
            "iterations_per_s": 1e3 / res["ms_per_step"],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
