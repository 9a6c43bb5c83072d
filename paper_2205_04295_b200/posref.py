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
