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
