"""Complex 2D field primitives (drop-in for ptychokit.fields).

Mirrors /root/reference/pkg/src/ptychokit/fields.py.  ``Geometry``, ``CropBox``
and ``sample_pixel_size`` are unchanged host metadata (fields.py:18-60).
``propagate`` (fields.py:71-84) and ``subpixel_shift`` (fields.py:110-122) run
on the GPU through ``pty_fft2``: numpy inputs are computed in float64 and
returned as numpy complex128 (reference semantics); torch CUDA inputs keep
their dtype and device.  ``crop``/``paste_add*`` (fields.py:87-107) are
device slicing; inside ``sweep`` they are fused into the sweep kernel.

B200 restriction: windows are powers of two in [16, 512] (the radix kernels);
other even sizes raise ShapeError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import BoundsError, GeometryError, ShapeError


def sample_pixel_size(wavelength: float, distance: float, window: int,
                      detector_pixel: float) -> float:
    """Sample-plane pixel size of a far-field setup: lambda * z / (W * delta_D)."""
    if wavelength <= 0 or distance <= 0 or window <= 0 or detector_pixel <= 0:
        raise GeometryError("all geometry inputs must be strictly positive")
    return wavelength * distance / (window * detector_pixel)


@dataclass(frozen=True)
class Geometry:
    """Optical geometry of a far-field transmission setup (fields.py:26-44)."""
    wavelength: float
    distance: float
    detector_pixel: float
    window: int
    sample_pixel: float

    @classmethod
    def create(cls, wavelength: float, distance: float, detector_pixel: float,
               window: int) -> "Geometry":
        if window < 8 or window % 2 != 0:
            raise GeometryError(f"window must be even and >= 8, got {window}")
        delta_s = sample_pixel_size(wavelength, distance, window, detector_pixel)
        return cls(wavelength, distance, detector_pixel, int(window), delta_s)


@dataclass(frozen=True)
class CropBox:
    """Square window into an object canvas, anchored at its top-left pixel."""
    row: int
    col: int
    side: int

    def check_inside(self, canvas_shape) -> None:
        h, w = canvas_shape[-2], canvas_shape[-1]
        if (self.row < 0 or self.col < 0 or self.side <= 0
                or self.row + self.side > h or self.col + self.side > w):
            raise BoundsError(f"crop box {self.side}px at ({self.row},{self.col}) "
                              f"outside {h}x{w} canvas")


def check_window(w: int) -> None:
    if w not in _native.WINDOWS:
        raise ShapeError(f"the B200 kernels need a power-of-two window in "
                         f"{_native.WINDOWS}, got {w}")


def to_device(a, dtype=None):
    """numpy / torch -> contiguous CUDA tensor (complex128 for numpy input)."""
    t = _native.torch()
    if isinstance(a, t.Tensor):
        x = a.to(_native.device())
        if not x.is_complex():
            x = x.to(t.complex128 if x.dtype == t.float64 else t.complex64)
    else:
        x = t.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.complex128)).to(_native.device())
    if dtype is not None:
        x = x.to(dtype)
    return x.contiguous()


def as_field(a):
    """Validate a 2D field (fields.py:63-68); returns a CUDA tensor."""
    x = to_device(a)
    if x.ndim != 2:
        raise ShapeError(f"field must be 2D, got ndim={x.ndim}")
    return x


def _result(x, like):
    t = _native.torch()
    return x if isinstance(like, t.Tensor) else x.cpu().numpy()


def propagate_(x, direction: str = "forward"):
    """In-place centered unitary DFT of a (..., W, W) CUDA tensor."""
    if direction not in ("forward", "backward"):
        raise ValueError(f"direction must be 'forward' or 'backward', got {direction!r}")
    _native.fft2(x, inverse=direction == "backward", centered=True)
    return x


def propagate(field, direction: str = "forward", geometry: Geometry | None = None,
              kind: str = "farfield"):
    """fields.py:71-84 -- fftshift(fft2(ifftshift(f), norm="ortho")) (or ifft2).

    kind="fresnel" (extension, needs ``geometry``): forward = P(Q * f),
    backward = conj(Q) * P^-1(f), Q = fresnel_chirp(geometry); the outer
    detector-plane chirp is dropped exactly as the far-field prefactor is."""
    if direction not in ("forward", "backward"):
        raise ValueError(f"direction must be 'forward' or 'backward', got {direction!r}")
    if kind not in ("farfield", "fresnel"):
        raise ValueError(f"kind must be 'farfield' or 'fresnel', got {kind!r}")
    x = as_field(field)
    if x.shape[0] != x.shape[1]:
        raise ShapeError(f"propagate requires a square field, got {tuple(x.shape)}")
    check_window(x.shape[0])
    if isinstance(field, _native.torch().Tensor):
        x = x.clone()   # never transform the caller's tensor in place
    if kind == "fresnel":
        if geometry is None:
            raise ValueError("the Fresnel propagator needs the geometry")
        q = fresnel_chirp(geometry, x.dtype, x.device)
        if direction == "forward":
            x *= q
            propagate_(x, direction)
        else:
            propagate_(x, direction)
            x *= q.conj()
        return _result(x, field)
    propagate_(x, direction)
    return _result(x, field)


def crop(canvas, box: CropBox):
    """fields.py:87-91 -- copy of the box region."""
    box.check_inside(tuple(canvas.shape))
    out = canvas[box.row:box.row + box.side, box.col:box.col + box.side]
    return out.clone() if hasattr(out, "clone") else out.copy()


def paste_add(canvas, box: CropBox, delta):
    out = canvas.clone() if hasattr(canvas, "clone") else np.array(canvas, copy=True)
    paste_add_inplace(out, box, delta)
    return out


def paste_add_inplace(canvas, box: CropBox, delta) -> None:
    """fields.py:101-107."""
    box.check_inside(tuple(canvas.shape))
    if tuple(delta.shape) != (box.side, box.side):
        raise ShapeError(f"delta shape {tuple(delta.shape)} != box side {box.side}")
    canvas[box.row:box.row + box.side, box.col:box.col + box.side] += delta


def fresnel_chirp(geometry: Geometry, dtype=None, device=None):
    """Quadratic phase of the single-FFT Fresnel regime (extension; the
    reference is far field only):
        Q[r, c] = exp(i pi ds^2 ((r - W/2)^2 + (c - W/2)^2) / (lambda z)),
    ds = geometry.sample_pixel.  The detector wave is Q2 * FFT(Q * psi); Q2 has
    unit modulus and the modulus constraint only uses |.| and the exact inverse,
    so a Fresnel reconstruction is the far-field one with the exit wave (hence
    the probe frame) multiplied by Q."""
    t = _native.torch()
    w = geometry.window
    k = np.pi * geometry.sample_pixel ** 2 / (geometry.wavelength * geometry.distance)
    r = np.arange(w, dtype=np.float64) - w // 2
    q = np.exp(1j * k * (r[:, None] ** 2 + r[None, :] ** 2))
    x = t.from_numpy(q)
    if device is not None or dtype is not None:
        x = x.to(device=device if device is not None else "cpu", dtype=dtype if dtype is not None else x.dtype)
    return x


def fourier_ramp(h: int, w: int, dx, dy, device, dtype):
    """exp(-2 pi i (fy dy + fx dx)) on the uncentered grid (fields.py:120-121).
    dx, dy: scalars or (B,) tensors -> (B, h, w)."""
    t = _native.torch()
    fy = t.fft.fftfreq(h, dtype=t.float64, device=device)[:, None]
    fx = t.fft.fftfreq(w, dtype=t.float64, device=device)[None, :]
    dx = t.as_tensor(dx, dtype=t.float64, device=device).reshape(-1, 1, 1)
    dy = t.as_tensor(dy, dtype=t.float64, device=device).reshape(-1, 1, 1)
    ramp = t.exp(-2j * np.pi * (fy * dy + fx * dx))
    return ramp.to(dtype)


def subpixel_shift(field, dx: float, dy: float):
    """fields.py:110-122 -- circular shift by (dy, dx) through a Fourier ramp."""
    x = as_field(field).clone()
    h, w = x.shape
    if abs(dy) >= h / 2 or abs(dx) >= w / 2:
        raise ShapeError(f"shift ({dy},{dx}) must satisfy |d| < side/2")
    check_window(h)
    _native.fft2(x, inverse=False, centered=False)
    x *= fourier_ramp(h, w, dx, dy, x.device, x.dtype)[0]
    _native.fft2(x, inverse=True, centered=False)
    return _result(x, field)
