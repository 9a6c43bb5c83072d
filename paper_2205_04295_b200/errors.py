"""Exception taxonomy of the drop-in (same names and bases as the reference's
/root/reference/pkg/src/ptychokit/errors.py:4-41), plus the mapping from the
C-ABI status word (include/ptycho_b200.h, ``PTY_ERR_*``) onto these classes."""


class PtychoError(Exception):
    """Base class for all toolkit errors."""


class GeometryError(PtychoError, ValueError):
    """Invalid optical geometry (non-positive length, bad window size)."""


class ShapeError(PtychoError, ValueError):
    """Array shape does not satisfy an operation's contract."""


class BoundsError(PtychoError, IndexError):
    """Crop box extends outside the canvas."""


class DegenerateInputError(PtychoError, ValueError):
    """Input carries no usable signal (all-zero field, flat crop)."""


class ParameterError(PtychoError, ValueError):
    """Configuration or algorithm parameter out of its valid range."""


class DataError(PtychoError, ValueError):
    """Measured data violates a physical precondition (e.g. negative intensity)."""


class PlanError(PtychoError, ValueError):
    """Scan plan cannot be realised (step/jitter would leave the canvas)."""


class DatasetIOError(PtychoError, IOError):
    """Dataset container on disk is missing, truncated or inconsistent."""


class BenchmarkRegression(PtychoError, AssertionError):
    """Timing harness detected the fast path losing to the reference path."""


class NativeError(PtychoError, RuntimeError):
    """The CUDA library failed (launch error, missing device, bad argument)."""


# status bits written by the kernels (include/ptycho_b200.h)
PTY_OK = 0
PTY_ERR_BOUNDS = 1 << 0          # crop box outside canvas       -> BoundsError
PTY_ERR_PROBE_ZERO = 1 << 1      # max sum_m |P_m|^2 == 0         -> DegenerateInputError
PTY_ERR_OBJECT_ZERO = 1 << 2     # max |o_j|^2 == 0 (probe update) -> DegenerateInputError
PTY_ERR_NEGATIVE_I = 1 << 3      # a measured intensity < 0      -> DataError
PTY_ERR_ARGUMENT = 1 << 8        # host-side argument check failed -> ParameterError/ShapeError
PTY_ERR_CUDA = 1 << 9            # CUDA runtime error              -> NativeError


def raise_for_status(status: int, where: str = "") -> None:
    """Translate a C-ABI status word into the reference's exception classes."""
    if status == PTY_OK:
        return
    tag = f" ({where})" if where else ""
    if status & PTY_ERR_NEGATIVE_I:
        raise DataError("measured intensities must be non-negative" + tag)
    if status & PTY_ERR_BOUNDS:
        raise BoundsError("crop box outside the object canvas" + tag)
    if status & PTY_ERR_PROBE_ZERO:
        raise DegenerateInputError("all probe modes are zero" + tag)
    if status & PTY_ERR_OBJECT_ZERO:
        raise DegenerateInputError("object crop is identically zero" + tag)
    if status & PTY_ERR_ARGUMENT:
        raise ParameterError("invalid argument to the CUDA library" + tag)
    raise NativeError(f"CUDA library status 0x{status:x}" + tag)
