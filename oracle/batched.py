"""Batched (semi-parallel) rPIE -- TEST INFRASTRUCTURE ONLY, parity UNPINNED.

The reference has no batched mode (engine.py:191 is strictly
sequential).  This module is the CPU statement of the extension the B200 build
adds, written so that batch size 1 reproduces the
reference sweep (engine.py:173-243) bit for bit:

  for each batch = contiguous slice of the visit order (engine.py:177-181):
    every position k in the batch sees the batch-start object and probes;
    object numerator  sum_k sum_m (psi'_km - P_m o_k) conj(P_m)      (engine.py:130-131)
    object denominator sum_k [gamma max sum|P|^2 + (1-gamma) sum|P|^2] (engine.py:135)
    probe numerator   sum_k alpha_P (psi'_km - P_m o_k) conj(o_k)     (engine.py:150)
    probe denominator sum_k [beta max|o_k|^2 + (1-beta)|o_k|^2]        (engine.py:148)
  then o <- o + ((o + alpha_O num/(den + eps max den)) - o) on covered pixels
       P <- P + num_P/(den_P + eps max den_P)

The sums are additive over positions, so a batch split across ranks is the sum
of per-rank ``contrib`` results (``apply`` after an all-reduce) -- the
decomposition tests/test_distributed_cpu.py checks with gloo.

Position refinement senses o_k (batch start) against the crop of the
updated object before the paste-add rounding (the reference's new_o_j,
engine.py:216,227).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import rpie


@dataclass
class Contrib:
    onum: np.ndarray          # canvas-shaped object numerator
    oden: np.ndarray          # canvas-shaped object denominator
    pnum: list                # per-mode probe numerators
    pden: np.ndarray          # probe denominator
    err_num: float
    err_den: float
    crops: list               # (j, r, c, o_j) for the sensors


def contrib(st: rpie.OracleState, patterns, window: int, cfg, ids) -> Contrib:
    """Update terms of the positions ``ids`` against the current state."""
    r0, c0 = st.canvas_origin
    rdt = rpie.real_dtype(st.obj.dtype)
    eps_rel = cfg.epsilon_rel
    update_probe = cfg.update_probe_modes and cfg.alpha_probe > 0
    out = Contrib(np.zeros_like(st.obj), np.zeros(st.obj.shape, dtype=rdt),
                  [np.zeros_like(p) for p in st.probes], np.zeros(st.probes[0].shape, dtype=rdt),
                  0.0, 0.0, [])
    power = np.zeros(st.probes[0].shape, dtype=rdt)
    for p in st.probes:
        power += np.abs(p) ** 2
    top = power.max()
    if top == 0.0:
        raise ZeroDivisionError("all probe modes are zero")
    for j in ids:
        r, c = (a - b for a, b in zip(rpie.anchor(st.positions[j]), (r0, c0)))
        o_j = st.obj[r:r + window, c:c + window].copy()
        i_j = patterns[j]
        corrected, _, total = rpie.modulus_project(st.probes, o_j, i_j, eps_rel)
        out.err_num += float(np.sum((np.sqrt(total) - np.sqrt(i_j.astype(rdt))) ** 2, dtype=np.float64))
        out.err_den += float(np.sum(i_j, dtype=np.float64))
        acc = np.zeros_like(o_j)
        for p, cw in zip(st.probes, corrected):
            acc += (cw - p * o_j) * np.conj(p)
        out.onum[r:r + window, c:c + window] += acc
        out.oden[r:r + window, c:c + window] += cfg.gamma * top + (1 - cfg.gamma) * power
        if update_probe:
            opow = np.abs(o_j) ** 2
            omax = opow.max()
            if omax == 0.0:
                raise ZeroDivisionError("object crop is identically zero")
            for m, (p, cw) in enumerate(zip(st.probes, corrected)):
                out.pnum[m] += cfg.alpha_probe * (cw - p * o_j) * np.conj(o_j)
            out.pden += cfg.beta * omax + (1 - cfg.beta) * opow
        out.crops.append((j, r, c, o_j, total))
    return out


def apply(st: rpie.OracleState, cfg, terms: Contrib) -> np.ndarray:
    """Apply summed update terms; returns the updated object before the paste
    rounding (the sensors' second input)."""
    eps_rel = cfg.epsilon_rel
    covered = terms.oden > 0
    dmax = terms.oden.max()
    upd = st.obj + cfg.alpha_obj * terms.onum / np.where(covered, terms.oden + eps_rel * dmax, 1)
    upd = np.where(covered, upd, st.obj)
    st.obj = np.where(covered, st.obj + (upd - st.obj), st.obj)
    if cfg.update_probe_modes and cfg.alpha_probe > 0:
        pd = terms.pden + eps_rel * terms.pden.max()
        st.probes = [p + q / pd for p, q in zip(st.probes, terms.pnum)]
    return upd


def sweep_batched(st: rpie.OracleState, patterns, window: int, cfg, batch: int,
                  order=None) -> rpie.OracleState:
    n = patterns.shape[0]
    if order is None:
        order = rpie.visit_order(n, cfg.position_order, cfg.shuffle_seed, st.iteration)
    pc = cfg.posref
    engaged = pc is not None and st.iteration >= pc.warmup_iterations
    bounds = rpie.position_bounds(st.obj.shape, st.canvas_origin, window)
    num = den = 0.0
    for s in range(0, n, batch):
        terms = contrib(st, patterns, window, cfg, order[s:s + batch])
        num += terms.err_num
        den += terms.err_den
        upd = apply(st, cfg, terms)
        if engaged:
            for j, r, c, o_j, total in terms.crops:
                after = upd[r:r + window, c:c + window]
                gx, gy, ok = rpie.sense(pc, o_j, after, total, patterns[j])
                if ok:
                    d = rpie.adam_update(st.adam_m, st.adam_v, st.adam_t, j, (gx, gy), pc)
                    rpie.clamp_move(st.positions, j, d, bounds)
    if (cfg.ortho_interval > 0 and len(st.probes) > 1
            and (st.iteration + 1) % cfg.ortho_interval == 0):
        st.probes = rpie.orthogonalize(st.probes)
    st.error_trace.append(num / max(den, rpie.TINY64))
    return st
