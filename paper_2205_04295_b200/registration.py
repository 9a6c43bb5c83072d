"""Batched subpixel registration on the GPU (drop-in for ptychokit.registration).

Guizar-Sicairos single-step upsampled-DFT registration, restated from
/root/reference/pkg/src/ptychokit/registration.py:43-128 as one batched
pipeline (``pty_register_batch``): cross-power spectrum (uncentered FFTs),
coarse argmax with the reference tie-break, and the floor(1.5 kappa)|odd-point
upsampled DFT around it.  Sign convention as the reference
(registration.py:9-12): the estimate is ADDED to the moving image.

numpy inputs are registered in float64 (reference precision); complex64 /
float32 torch inputs use the fp32 kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import DegenerateInputError, ParameterError, ShapeError
from .fields import check_window

PHASE_EPS_REL = 1e-12


@dataclass(frozen=True)
class ShiftEstimate:
    dy: float
    dx: float
    peak_value: float
    upsample: int


def _kappa(upsample) -> int:
    k = int(upsample)
    if not (k == 1 or 2 <= k <= 1000):
        raise ParameterError(f"upsample factor must be in [1, 1000], got {k}")
    return k


def _weighting(w: str) -> int:
    if w == "phase":
        return 0
    if w == "raw":
        return 1
    raise ParameterError(f"weighting must be 'phase' or 'raw', got {w!r}")


def register_batch(refs, movs, weighting: str = "phase", upsample: int = 1):
    """Register n pairs; refs/movs are (n, W, W) arrays or tensors.

    Returns (dy, dx, peak, ok) as float64/int32 CUDA tensors; ok = 0 marks a
    pair whose cross-power spectrum is identically zero."""
    t = _native.torch()
    kappa = _kappa(upsample)
    wcode = _weighting(weighting)
    use64 = not isinstance(refs, t.Tensor) or refs.dtype in (t.complex128, t.float64)
    cdt = t.complex128 if use64 else t.complex64
    dev = _native.device()

    def dev_of(a):
        return (a.to(dev) if isinstance(a, t.Tensor)
                else t.from_numpy(np.ascontiguousarray(a)).to(dev))

    r, m = dev_of(refs), dev_of(movs)
    if r.shape != m.shape or r.ndim != 3 or r.shape[-1] != r.shape[-2]:
        raise ShapeError(f"need equal square shapes, got {tuple(r.shape)} vs {tuple(m.shape)}")
    n, w = r.shape[0], r.shape[-1]
    check_window(w)
    work = t.empty((n, 2, w, w), dtype=cdt, device=dev)
    work[:, 0] = r.to(cdt)
    work[:, 1] = m.to(cdt)
    dy = t.empty(n, dtype=t.float64, device=dev)
    dx = t.empty_like(dy)
    peak = t.empty_like(dy)
    ok = t.empty(n, dtype=t.int32, device=dev)
    _native.register_batch(work, w, n, wcode, kappa, dy, dx, peak, ok)
    return dy, dx, peak, ok


# --------------------------------------- the pipeline's steps, one call each --
# registration.py:43-120 as separate GPU calls (pty_cross_power_spectrum,
# pty_coarse_argmax, pty_upsampled_idft, pty_argmax_abs) for callers that
# compose them; register() runs the fused batched pipeline instead.

def _is_tensor(a) -> bool:
    return isinstance(a, _native.torch().Tensor)


def _pair(reference, moving):
    """registration.py:35-40 -- equal square fields (complex; real inputs promoted)."""
    t = _native.torch()
    ref = reference if _is_tensor(reference) else np.asarray(reference)
    mov = moving if _is_tensor(moving) else np.asarray(moving)
    if ref.ndim != 2 or tuple(ref.shape) != tuple(mov.shape) or ref.shape[0] != ref.shape[1]:
        raise ShapeError(f"need equal square shapes, got {tuple(ref.shape)} vs {tuple(mov.shape)}")
    check_window(int(ref.shape[0]))
    use32 = any(_is_tensor(a) and a.dtype in (t.complex64, t.float32) for a in (ref, mov))
    cdt = t.complex64 if use32 else t.complex128
    dev = _native.device()

    def up(a):
        x = a if _is_tensor(a) else t.from_numpy(np.ascontiguousarray(a))
        return x.to(dev).to(cdt)
    return up(ref), up(mov)


def cross_power_spectrum(reference, moving, weighting: str = "phase"):
    """registration.py:43-56 -- F(ref) * conj(F(mov)) (uncentered), whitened
    to unit magnitude for "phase"; DegenerateInputError if identically zero."""
    t = _native.torch()
    ref, mov = _pair(reference, moving)
    w = ref.shape[-1]
    wcode = 1 if weighting not in ("phase", "raw") else _weighting(weighting)
    work = t.empty((1, 2, w, w), dtype=ref.dtype, device=ref.device)
    work[0, 0] = ref
    work[0, 1] = mov
    xps = t.empty((1, w, w), dtype=ref.dtype, device=ref.device)
    ok = t.empty(1, dtype=t.int32, device=ref.device)
    _native.cross_power_spectrum(work, w, 1, wcode, xps, ok)
    if int(ok.item()) == 0:
        raise DegenerateInputError("cross-power spectrum is identically zero")
    _weighting(weighting)                         # registration.py:56: checked after the spectrum
    out = xps[0]
    return out if _is_tensor(reference) else out.cpu().numpy()


def _signed(index: int, side: int) -> int:
    """registration.py:59-64."""
    v = index - side // 2
    if v <= -side // 2 and side % 2 == 0:
        v += side
    return v


def coarse_shift(xps) -> ShiftEstimate:
    """registration.py:67-81 -- argmax of |ifft2(xps)| over signed lags, ties
    broken toward zero shift (min |dy|+|dx|, then dy, then dx)."""
    t = _native.torch()
    x, _ = _pair(xps, xps)
    corr = x.clone()[None]
    _native.fft2(corr, inverse=True, centered=False)
    vals = t.empty(3, dtype=t.float64, device=x.device)
    _native.coarse_argmax(corr, vals[0:1], vals[1:2], vals[2:3])
    dy, dx, peak = vals.cpu().numpy()
    return ShiftEstimate(float(dy), float(dx), float(peak), 1)


def upsampled_idft(xps, rows, cols):
    """registration.py:84-96 -- inverse DFT of xps at fractional (row, col)
    lags by two explicit DFT-matrix products (no zero padding)."""
    t = _native.torch()
    x, _ = _pair(xps, xps)
    dev = x.device
    r = t.as_tensor(np.asarray(rows, np.float64).reshape(-1), device=dev)
    c = t.as_tensor(np.asarray(cols, np.float64).reshape(-1), device=dev)
    out = t.empty((r.numel(), c.numel()), dtype=x.dtype, device=dev)
    _native.upsampled_idft(x, r, c, out)
    return out if _is_tensor(xps) else out.cpu().numpy()


def _refine_offsets(kappa: int) -> np.ndarray:
    """registration.py:99-105 -- odd point count <= 1.5 kappa + 1."""
    n = int(np.floor(1.5 * kappa))
    if n % 2 == 0:
        n += 1
    half = n // 2
    return np.arange(-half, half + 1) / kappa


def refine_shift(xps, coarse: ShiftEstimate, kappa: int) -> ShiftEstimate:
    """registration.py:108-120 -- refine a coarse shift to 1/kappa pixel on a
    local upsampled-DFT grid (first maximum in row-major order)."""
    t = _native.torch()
    kappa = int(kappa)
    if kappa == 1:
        return coarse
    if not 2 <= kappa <= 1000:
        raise ParameterError(f"upsample factor must be in [1, 1000], got {kappa}")
    offs = _refine_offsets(kappa)
    rows = coarse.dy + offs
    cols = coarse.dx + offs
    x, _ = _pair(xps, xps)
    corr = upsampled_idft(x, rows, cols)
    idx = t.empty(1, dtype=t.int64, device=x.device)
    val = t.empty(1, dtype=t.float64, device=x.device)
    _native.argmax_abs(corr, idx, val)
    iy, ix = divmod(int(idx.item()), len(cols))
    return ShiftEstimate(float(rows[iy]), float(cols[ix]), float(val.item()), kappa)


def register(reference, moving, weighting: str = "phase", upsample: int = 1) -> ShiftEstimate:
    """registration.py:123-128 for one pair."""
    t = _native.torch()
    ref = reference if isinstance(reference, t.Tensor) else np.asarray(reference)
    mov = moving if isinstance(moving, t.Tensor) else np.asarray(moving)
    if ref.ndim != 2 or tuple(ref.shape) != tuple(mov.shape) or ref.shape[0] != ref.shape[1]:
        raise ShapeError(f"need equal square shapes, got {tuple(ref.shape)} vs {tuple(mov.shape)}")
    if isinstance(ref, t.Tensor):
        ref, mov = ref[None], mov[None]
    else:
        ref = np.asarray(ref, np.complex128)[None]
        mov = np.asarray(mov, np.complex128)[None]
    dy, dx, peak, ok = register_batch(ref, mov, weighting, upsample)
    vals = t.stack([dy, dx, peak, ok.double()]).cpu().numpy()[:, 0]
    if vals[3] == 0:
        raise DegenerateInputError("cross-power spectrum is identically zero")
    return ShiftEstimate(float(vals[0]), float(vals[1]), float(vals[2]), _kappa(upsample))
