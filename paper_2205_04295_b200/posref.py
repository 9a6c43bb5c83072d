"""Adam-driven scan-position refinement: configuration and per-position state.

Drop-in for /root/reference/pkg/src/ptychokit/posref.py.  ``PosRefConfig``
keeps the reference's fields, defaults and validation (posref.py:22-39).
``AdamBuffers`` keeps the reference layout (m, v: (N, 2) float64; t: (N,)
int64, posref.py:42-54) but lives in HBM: the Adam recurrence
(posref.py:87-99) and the clamp (posref.py:102-113) run as one float64 CUDA
kernel over every sensed position after the sweep's registration batch
(``pty_adam_apply`` in include/ptycho_b200.h).

The sensors (posref.py:57-84) are fused into the sweep: XCORR_A registers each
position's pre-update object crop against its update, XCORR_B the modelled
against the measured intensity; both feed the batched Guizar-Sicairos kernel
(registration.py in this package).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native


@dataclass(frozen=True)
class PosRefConfig:
    sensor: str = "XCORR_A"       # XCORR_A | XCORR_B
    step_size: float = 0.5        # pixels per unit surrogate gradient (Adam lr)
    beta1: float = 0.9
    beta2: float = 0.999
    eps_adam: float = 1e-8
    warmup_iterations: int = 10
    kappa: int = 100              # registration upsample factor
    max_correction: float = 1.0   # per-iteration clip, pixels

    def __post_init__(self) -> None:
        if not (0 < self.beta1 < 1 and 0 < self.beta2 < 1):
            raise ValueError("beta1 and beta2 must lie in (0, 1)")
        if self.step_size <= 0:
            raise ValueError("step_size must be positive")
        if self.sensor not in ("XCORR_A", "XCORR_B"):
            raise ValueError(f"unknown sensor {self.sensor!r}")


class AdamBuffers:
    """Per-position first/second moments and step counts, resident on the GPU."""

    def __init__(self, m, v, t):
        self.m = m   # torch float64 (N, 2)
        self.v = v   # torch float64 (N, 2)
        self.t = t   # torch int64 (N,)

    @classmethod
    def zeros(cls, n_positions: int, device=None) -> "AdamBuffers":
        torch = _native.torch()
        dev = device if device is not None else _native.device()
        return cls(m=torch.zeros((n_positions, 2), dtype=torch.float64, device=dev),
                   v=torch.zeros((n_positions, 2), dtype=torch.float64, device=dev),
                   t=torch.zeros(n_positions, dtype=torch.int64, device=dev))

    def numpy(self):
        return (self.m.cpu().numpy(), self.v.cpu().numpy(), self.t.cpu().numpy())


def adam_apply(positions, buffers: AdamBuffers, gx, gy, ok, config: PosRefConfig,
               bounds, index=None) -> None:
    """Adam step + clamp for every position with ok != 0 (posref.py:87-113).

    ``gx, gy`` (float64) and ``ok`` (int32) are device tensors indexed like
    ``positions`` unless ``index`` (int32, device) maps sensed entries to
    position ids."""
    _native.adam_apply(positions, buffers, gx, gy, ok, config, bounds, index)


# ------------------------------------------- per-position public functions --
# posref.py:57-113 one position at a time, on the GPU (the sweep runs the same
# arithmetic batched over all sensed positions: adam_apply above).

def _sense(reference, moving, weighting: str, kappa: int):
    """posref.py:57-63 -- (gx, gy, confident); a degenerate spectrum is not confident."""
    from .errors import DegenerateInputError
    from .registration import register
    try:
        est = register(reference, moving, weighting=weighting, upsample=kappa)
    except DegenerateInputError:
        return 0.0, 0.0, False
    return est.dx, est.dy, True


def sense_shift_A(crop_before, crop_after, kappa: int):
    """posref.py:66-76 -- object crop vs its update, raw weighting."""
    return _sense(crop_before, crop_after, "raw", kappa)


def sense_shift_B(intensity_model, intensity_measured, kappa: int):
    """posref.py:79-84 -- modelled vs measured intensity (real), raw weighting."""
    torch = _native.torch()

    def real(a):
        if isinstance(a, torch.Tensor):
            return a.real if a.is_complex() else a
        return np.asarray(a, float)
    return _sense(real(intensity_model), real(intensity_measured), "raw", kappa)


def adam_step(buffers: AdamBuffers, j: int, g, config: PosRefConfig):
    """posref.py:87-99 -- one Adam update of position j (float64 on the GPU);
    returns the clipped (dx, dy)."""
    torch = _native.torch()
    delta = torch.empty(2, dtype=torch.float64, device=buffers.m.device)
    gx, gy = (float(v) for v in g)
    _native.adam_step(buffers, int(j), gx, gy, config, delta)
    dx, dy = delta.cpu().numpy()
    return float(dx), float(dy)


def apply_correction(positions, j: int, delta, bounds) -> bool:
    """posref.py:102-113 -- add (dx, dy) to position j and clamp to
    (xmin, ymin, xmax, ymax); False when the clamp engaged.  ``positions`` is
    an (N, 2) float64 CUDA tensor (ReconState.positions) or numpy array
    (updated in place)."""
    torch = _native.torch()
    host = not isinstance(positions, torch.Tensor)
    pos = torch.from_numpy(np.ascontiguousarray(positions, np.float64)).to(_native.device()) if host \
        else positions
    inside = torch.empty(1, dtype=torch.int32, device=pos.device)
    _native.apply_correction(pos, int(j), float(delta[0]), float(delta[1]), bounds, inside)
    if host:
        positions[j] = pos[j].cpu().numpy()
    return bool(inside.item())
