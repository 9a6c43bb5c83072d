"""Numpy restatement of the reference rPIE sweep -- TEST INFRASTRUCTURE ONLY.

Restates, for the oracle, the semantics of
  /root/reference/pkg/src/ptychokit/fields.py   (propagate, crop/paste)
  /root/reference/pkg/src/ptychokit/engine.py   (initialize, magnitude_correct,
                                                update_object/probe, sweep)
  /root/reference/pkg/src/ptychokit/posref.py   (sensors, Adam, clamp)
Each function names the file:line range it follows.  ``cdt`` selects the
complex dtype: complex128 reproduces the reference; complex64 is the
single-precision shadow used to bound the fp32 CUDA kernels.

Parity pin: tests/test_oracle_golden.py checks this module against vectors
produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import registration as oreg

TINY64 = np.finfo(np.float64).tiny


def real_dtype(cdt):
    return np.float32 if np.dtype(cdt) == np.complex64 else np.float64


# ------------------------------------------------------------------ fields --

def centered_fft2(f: np.ndarray, inverse: bool = False) -> np.ndarray:
    """fields.py:71-84 -- unitary centered 2D DFT, fftshift(fft2(ifftshift))."""
    g = np.fft.ifftshift(f)
    g = np.fft.ifft2(g, norm="ortho") if inverse else np.fft.fft2(g, norm="ortho")
    return np.fft.fftshift(g)


def anchor(pos_xy) -> tuple[int, int]:
    """engine.py:69-70 -- (row, col) = (round(y), round(x)), half-to-even."""
    return int(round(float(pos_xy[1]))), int(round(float(pos_xy[0])))


def box_inside(row: int, col: int, side: int, shape) -> bool:
    """fields.py:55-60 -- CropBox.check_inside."""
    h, w = shape
    return not (row < 0 or col < 0 or row + side > h or col + side > w)


# ------------------------------------------------------------------- state --

@dataclass
class OracleState:
    """Mirror of engine.ReconState (engine.py:53-66) with plain arrays."""
    obj: np.ndarray
    probes: list
    positions: np.ndarray
    canvas_origin: tuple
    adam_m: np.ndarray | None = None
    adam_v: np.ndarray | None = None
    adam_t: np.ndarray | None = None
    error_trace: list = field(default_factory=list)
    modulus_error_trace: list = field(default_factory=list)

    @property
    def iteration(self) -> int:
        return len(self.error_trace)

    def copy(self) -> "OracleState":
        c = lambda a: None if a is None else np.array(a, copy=True)
        return OracleState(self.obj.copy(), [p.copy() for p in self.probes],
                           self.positions.copy(), tuple(self.canvas_origin),
                           c(self.adam_m), c(self.adam_v), c(self.adam_t),
                           list(self.error_trace), list(self.modulus_error_trace))


def initialize(patterns, positions, window: int, cfg, cdt=np.complex128, chirp=None) -> OracleState:
    """engine.py:73-101.

    canvas = anchor bounding box + window, unit transmission; mode 1 is the
    back-propagated mean amplitude; mode p>1 is mode 1 times complex noise from
    default_rng([init_seed, p]), Gram-Schmidt'ed, scaled to 1% of mode-1 power.
    """
    anchors = np.array([anchor(p) for p in positions], dtype=np.int64)
    origin = anchors.min(axis=0)
    extent = anchors.max(axis=0) - origin + window
    obj = np.ones((int(extent[0]), int(extent[1])), dtype=cdt)
    amp = np.sqrt(np.maximum(np.asarray(patterns, np.float64).mean(axis=0), 0.0))
    first = centered_fft2(amp.astype(np.complex128), inverse=True)
    modes = [first]
    first_power = np.sum(np.abs(first) ** 2)
    for p in range(1, cfg.mode_count):
        rng = np.random.default_rng([cfg.init_seed, p])
        noise = rng.standard_normal((window, window)) + 1j * rng.standard_normal((window, window))
        cand = first * noise
        for prev in modes:
            cand = cand - prev * (np.vdot(prev, cand) / np.vdot(prev, prev))
        cand *= np.sqrt(0.01 * first_power / np.sum(np.abs(cand) ** 2))
        modes.append(cand)
    if chirp is not None:   # Fresnel extension: back-propagation ends with conj(Q)
        modes = [np.conj(chirp) * m for m in modes]
    st = OracleState(obj=obj, probes=[m.astype(cdt) for m in modes],
                     positions=np.array(positions, dtype=np.float64, copy=True),
                     canvas_origin=(int(origin[0]), int(origin[1])))
    if cfg.posref is not None:
        n = len(positions)
        st.adam_m = np.zeros((n, 2))
        st.adam_v = np.zeros((n, 2))
        st.adam_t = np.zeros(n, dtype=np.int64)
    return st


# ------------------------------------------------------------- one visit --

def fresnel_chirp(geometry):
    """Single-FFT Fresnel regime (extension, not in the reference): the exit
    wave is multiplied by Q = exp(i pi ds^2 |x|^2 / (lambda z)) before the
    centered FFT and by conj(Q) after the inverse (the detector-plane chirp
    drops out of |.|, like the far-field prefactor, fields.py:4-6)."""
    w = geometry.window
    k = np.pi * geometry.sample_pixel ** 2 / (geometry.wavelength * geometry.distance)
    r = np.arange(w, dtype=np.float64) - w // 2
    return np.exp(1j * k * (r[:, None] ** 2 + r[None, :] ** 2))


def modulus_project(probes, o_j, i_j, eps_rel=1e-12, chirp=None):
    """engine.py:104-120 -- mixed-state modulus constraint.

    Returns (corrected exit waves, detector waves, total detector intensity).
    ``chirp``: optional Fresnel quadratic phase (extension)."""
    if np.any(i_j < 0):
        raise ValueError("negative intensity")  # DataError in the reference
    rdt = real_dtype(o_j.dtype)
    if chirp is not None:
        det = [centered_fft2(chirp * p * o_j) for p in probes]
    else:
        det = [centered_fft2(p * o_j) for p in probes]
    total = np.zeros(i_j.shape, dtype=rdt)
    for d in det:
        total += np.abs(d) ** 2
    eps = eps_rel * max(float(total.max()), TINY64)
    if rdt == np.float32:
        eps = np.float32(eps_rel) * max(np.float32(total.max()), np.finfo(np.float32).tiny)
    ratio = np.sqrt(i_j.astype(rdt)) / np.sqrt(total + eps)
    corrected = [centered_fft2(ratio * d, inverse=True) for d in det]
    if chirp is not None:
        corrected = [np.conj(chirp) * c for c in corrected]
    return corrected, det, total


def object_step(o_j, probes, corrected, alpha_obj, gamma, eps_rel=1e-12):
    """engine.py:123-137 -- rPIE object update (gamma = 1: ePIE)."""
    rdt = real_dtype(o_j.dtype)
    acc = np.zeros_like(o_j)
    power = np.zeros(o_j.shape, dtype=rdt)
    for p, c in zip(probes, corrected):
        acc += (c - p * o_j) * np.conj(p)
        power += np.abs(p) ** 2
    top = power.max()
    if top == 0.0:
        raise ZeroDivisionError("all probe modes are zero")  # DegenerateInputError
    den = gamma * top + (1 - gamma) * power
    den = den + eps_rel * den.max()
    return o_j + alpha_obj * acc / den


def probe_step(probe, o_j, corrected, alpha_probe, beta, eps_rel=1e-12):
    """engine.py:140-150 -- rPIE probe update for one mode (beta = 1: ePIE)."""
    power = np.abs(o_j) ** 2
    top = power.max()
    if top == 0.0:
        raise ZeroDivisionError("object crop is identically zero")
    den = beta * top + (1 - beta) * power
    den = den + eps_rel * den.max()
    return probe + alpha_probe * (corrected - probe * o_j) * np.conj(o_j) / den


def orthogonalize(probes):
    """engine.py:153-164 -- power-preserving Gram-Schmidt, strongest first."""
    before = sum(np.sum(np.abs(p) ** 2) for p in probes)
    out = []
    for p in probes:
        q = p.copy()
        for prev in out:
            q -= prev * (np.vdot(prev, q) / np.vdot(prev, prev))
        out.append(q)
    after = sum(np.sum(np.abs(p) ** 2) for p in out)
    s = np.sqrt(before / after) if after > 0 else 1.0
    return [q * s for q in out]


# ------------------------------------------------------------ sweep plumbing --

def visit_order(n: int, position_order: str, shuffle_seed: int, iteration: int) -> np.ndarray:
    """engine.py:177-181."""
    if position_order == "shuffled":
        return np.random.default_rng([shuffle_seed, iteration]).permutation(n)
    return np.arange(n)


def position_bounds(obj_shape, origin, window):
    """engine.py:167-170 -> (xmin, ymin, xmax, ymax)."""
    h, w = obj_shape
    r0, c0 = origin
    return float(c0), float(r0), float(c0 + w - window), float(r0 + h - window)


def adam_update(m, v, t, j, g, pc):
    """posref.py:87-99 -- one Adam step for position j; returns clipped (dx, dy)."""
    g = np.asarray(g, float)
    t[j] += 1
    tj = t[j]
    m[j] = pc.beta1 * m[j] + (1 - pc.beta1) * g
    v[j] = pc.beta2 * v[j] + (1 - pc.beta2) * g * g
    mh = m[j] / (1 - pc.beta1 ** tj)
    vh = v[j] / (1 - pc.beta2 ** tj)
    d = pc.step_size * mh / (np.sqrt(vh) + pc.eps_adam)
    d = np.clip(d, -pc.max_correction, pc.max_correction)
    return float(d[0]), float(d[1])


def clamp_move(positions, j, delta, bounds):
    """posref.py:102-113 -- add (dx, dy) to position j and clamp to bounds."""
    xmin, ymin, xmax, ymax = bounds
    x = positions[j, 0] + delta[0]
    y = positions[j, 1] + delta[1]
    positions[j, 0] = min(max(x, xmin), xmax)
    positions[j, 1] = min(max(y, ymin), ymax)


def sense(pc, o_before, o_after, total, i_j):
    """posref.py:57-84 -- XCORR_A / XCORR_B sensors; returns (gx, gy, ok)."""
    if pc.sensor == "XCORR_A":
        ref, mov = o_before.astype(np.complex128), o_after.astype(np.complex128)
    else:
        ref = np.asarray(total, np.float64).astype(np.complex128)
        mov = np.asarray(i_j, np.float64).astype(np.complex128)
    try:
        est = oreg.register(ref, mov, "raw", pc.kappa)
    except oreg.Degenerate:
        return 0.0, 0.0, False
    return est.dx, est.dy, True


def subpixel_shift(f: np.ndarray, dx: float, dy: float) -> np.ndarray:
    """fields.py:110-122 -- circular shift by (dy, dx) through a Fourier phase ramp."""
    h, w = f.shape
    fy = np.fft.fftfreq(h)[:, None]
    fx = np.fft.fftfreq(w)[None, :]
    return np.fft.ifft2(np.fft.fft2(f) * np.exp(-2j * np.pi * (fy * dy + fx * dx)))


def sweep(st: OracleState, patterns, window: int, cfg, order=None, chirp=None) -> OracleState:
    """engine.py:173-243 -- one pass over every position, mutating ``st``.
    ``chirp``: Fresnel quadratic phase (extension; None = the reference).
    ``cfg.subpixel_gather`` (extension, parity unpinned): the crop is the
    simulator's extract_view (simulate.py:157-166) -- integer crop shifted by
    (-rx, -ry) -- and the object update is shifted back by (rx, ry) before the
    paste; a residual of exactly zero leaves the crop untouched."""
    subpixel = bool(getattr(cfg, "subpixel_gather", False))
    n = patterns.shape[0]
    if order is None:
        order = visit_order(n, cfg.position_order, cfg.shuffle_seed, st.iteration)
    pc = cfg.posref
    engaged = pc is not None and st.iteration >= pc.warmup_iterations
    bounds = position_bounds(st.obj.shape, st.canvas_origin, window)
    r0, c0 = st.canvas_origin
    rdt = real_dtype(st.obj.dtype)
    num = 0.0
    den = 0.0
    worst = 0.0
    for j in order:
        i_j = patterns[j]
        ar, ac = anchor(st.positions[j])
        r, c = ar - r0, ac - c0
        if not box_inside(r, c, window, st.obj.shape):
            raise IndexError(f"crop box at ({r},{c}) outside canvas")
        o_j = st.obj[r:r + window, c:c + window].copy()
        rx = float(st.positions[j, 0]) - ac
        ry = float(st.positions[j, 1]) - ar
        shifted = subpixel and (rx != 0.0 or ry != 0.0)
        if shifted:
            o_j = subpixel_shift(o_j, -rx, -ry).astype(st.obj.dtype)
        corrected, det, _ = modulus_project(st.probes, o_j, i_j, cfg.epsilon_rel, chirp)
        total = np.zeros(i_j.shape, dtype=rdt)
        for d in det:
            total += np.abs(d) ** 2
        num += float(np.sum((np.sqrt(total) - np.sqrt(i_j.astype(rdt))) ** 2, dtype=np.float64))
        den += float(np.sum(i_j, dtype=np.float64))
        if cfg.track_modulus_error:
            after = np.zeros(i_j.shape, dtype=rdt)
            for cw in corrected:
                after += np.abs(centered_fft2(cw)) ** 2
            guard = total > 1e-3 * total.max()
            if np.any(guard):
                rel = np.abs(after[guard] - i_j[guard]) / np.maximum(i_j[guard], TINY64)
                worst = max(worst, float(rel.max()))
        new_o = object_step(o_j, st.probes, corrected, cfg.alpha_obj, cfg.gamma,
                            cfg.epsilon_rel)
        if cfg.update_probe_modes and cfg.alpha_probe > 0:
            st.probes = [probe_step(p, o_j, cw, cfg.alpha_probe, cfg.beta, cfg.epsilon_rel)
                         for p, cw in zip(st.probes, corrected)]
        delta = new_o - o_j
        if shifted:
            delta = subpixel_shift(delta, rx, ry).astype(st.obj.dtype)
        st.obj[r:r + window, c:c + window] += delta
        if engaged:
            gx, gy, ok = sense(pc, o_j, new_o, total, i_j)
            if ok:
                d = adam_update(st.adam_m, st.adam_v, st.adam_t, j, (gx, gy), pc)
                clamp_move(st.positions, j, d, bounds)
    if (cfg.ortho_interval > 0 and len(st.probes) > 1
            and (st.iteration + 1) % cfg.ortho_interval == 0):
        st.probes = orthogonalize(st.probes)
    st.error_trace.append(num / max(den, TINY64))
    if cfg.track_modulus_error:
        st.modulus_error_trace.append(worst)
    return st
