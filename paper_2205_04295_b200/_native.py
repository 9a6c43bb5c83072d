"""ctypes binding of libptycho_b200.so (the C ABI in include/ptycho_b200.h).

PyTorch is used only as the device allocator and stream provider: tensors are
passed as raw device pointers plus sizes.  There is no fallback: if the
library or a CUDA device is missing, every entry point raises NativeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import NativeError, raise_for_status

_PKG = Path(__file__).resolve().parent
_LIB_PATH = _PKG / "libptycho_b200.so"
_lock = threading.Lock()
_lib = None

DTYPE_C64 = 0
DTYPE_C128 = 1
SENSE_NONE, SENSE_XCORR_A, SENSE_XCORR_B = 0, 1, 2
MAX_SLOTS = 24
WINDOWS = (16, 32, 64, 128, 256, 512)


def torch():
    import torch as _t
    return _t


def device():
    t = torch()
    if not t.cuda.is_available():
        raise NativeError("no CUDA device visible: the B200 path has no CPU fallback")
    return t.device("cuda", t.cuda.current_device())


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


class PtySlot(C.Structure):
    _fields_ = [("obj", C.c_void_p), ("H", C.c_int32), ("Wc", C.c_int32),
                ("r0", C.c_int32), ("c0", C.c_int32), ("probes", C.c_void_p),
                ("patterns", C.c_void_p), ("patterns_t", C.c_void_p), ("positions", C.c_void_p),
                ("order", C.c_void_p), ("stage", C.c_void_p), ("err_out", C.c_void_p),
                ("status", C.c_void_p)]


class PtySweepArgs(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("window", C.c_int32), ("modes", C.c_int32),
                ("n_positions", C.c_int32), ("n_slots", C.c_int32),
                ("slots", C.POINTER(PtySlot)),
                ("alpha_obj", C.c_double), ("alpha_probe", C.c_double), ("beta", C.c_double),
                ("gamma", C.c_double), ("epsilon_rel", C.c_double),
                ("update_probe", C.c_int32), ("track_modulus", C.c_int32), ("sense", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64)]


class PtyBatchArgs(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("window", C.c_int32), ("modes", C.c_int32),
                ("n_positions", C.c_int32), ("obj", C.c_void_p), ("H", C.c_int32), ("Wc", C.c_int32),
                ("r0", C.c_int32), ("c0", C.c_int32), ("probes", C.c_void_p),
                ("patterns", C.c_void_p), ("patterns_t", C.c_void_p), ("positions", C.c_void_p),
                ("batch", C.c_void_p), ("n_batch", C.c_int32), ("visit0", C.c_int32),
                ("alpha_obj", C.c_double), ("alpha_probe", C.c_double), ("beta", C.c_double),
                ("gamma", C.c_double), ("epsilon_rel", C.c_double),
                ("update_probe", C.c_int32), ("track_modulus", C.c_int32), ("sense", C.c_int32),
                ("stage", C.c_void_p), ("obj_acc", C.c_void_p), ("probe_acc", C.c_void_p),
                ("err_part", C.c_void_p), ("status", C.c_void_p),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_int64)]


def _declare(lib):
    i32, i64, vp, dp = C.c_int32, C.c_int64, C.c_void_p, C.c_double
    sig = {
        "pty_abi_version": (C.c_int, []),
        "pty_launch_count": (i64, []),
        "pty_barrier_bench": (C.c_int, [i32, i32, C.POINTER(C.c_double)]),
        "pty_timeline": (i64, [vp, i64, C.POINTER(i32)]),
        "pty_device_info": (C.c_int, [C.POINTER(i32)] * 4),
        "pty_sweep_workspace_bytes": (i64, [i32] * 5),
        "pty_sweep": (C.c_int, [C.POINTER(PtySweepArgs), vp]),
        "pty_sweep_subpixel": (C.c_int, [C.POINTER(PtySweepArgs), vp]),
        "pty_fft2": (C.c_int, [vp, i32, i32, i32, i32, i32, vp]),
        "pty_register_batch": (C.c_int, [vp, vp, vp, i32, i32, i32, i32, i32, i32,
                                         vp, vp, vp, vp, vp, i64, vp]),
        "pty_register_scratch_bytes": (i64, [i32, i32, i32]),
        "pty_adam_apply": (C.c_int, [vp] * 8 + [i32] + [dp] * 9 + [vp]),
        "pty_init_probes": (C.c_int, [vp, i32, vp, i32, vp, i32, i32, vp, i64, vp]),
        "pty_orthogonalize": (C.c_int, [vp, i32, i32, i32, vp]),
        "pty_check_patterns": (C.c_int, [vp, i32, i64, vp, vp]),
        "pty_batch_workspace_bytes": (i64, [i32] * 6),
        "pty_batch_contrib": (C.c_int, [C.POINTER(PtyBatchArgs), vp]),
        "pty_batch_apply": (C.c_int, [C.POINTER(PtyBatchArgs), vp]),
        "pty_batch_finalize": (C.c_int, [vp, i32, i32, vp, vp]),
        "pty_accumulate": (C.c_int, [vp, vp, i64, i32, vp]),
        "pty_visit_scratch_bytes": (i64, [i32, i32, i32]),
        "pty_magnitude_correct": (C.c_int, [i32, i32, i32, vp, vp, vp, dp, vp, vp, vp, vp, i64, vp]),
        "pty_update_object": (C.c_int, [i32, i32, i32, vp, vp, vp, dp, dp, dp, vp, vp, vp, i64, vp]),
        "pty_update_probe": (C.c_int, [i32, i32, vp, vp, vp, dp, dp, dp, vp, vp, vp, i64, vp]),
        "pty_cross_power_spectrum": (C.c_int, [vp, vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, i64, vp]),
        "pty_coarse_argmax": (C.c_int, [vp, i32, i32, i32, vp, vp, vp, vp]),
        "pty_upsampled_idft_scratch_bytes": (i64, [i32, i32, i32]),
        "pty_upsampled_idft": (C.c_int, [vp, i32, i32, vp, i32, vp, i32, vp, vp, i64, vp]),
        "pty_argmax_abs": (C.c_int, [vp, i32, i64, vp, vp, vp]),
        "pty_adam_step": (C.c_int, [vp, vp, vp, i32, dp, dp, dp, dp, dp, dp, dp, vp, vp]),
        "pty_apply_correction": (C.c_int, [vp, i32, dp, dp, dp, dp, dp, dp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


EXPORTS = ("pty_abi_version", "pty_launch_count", "pty_barrier_bench", "pty_timeline", "pty_device_info", "pty_sweep_workspace_bytes", "pty_sweep", "pty_sweep_subpixel",
           "pty_fft2", "pty_register_batch", "pty_register_scratch_bytes", "pty_adam_apply",
           "pty_init_probes", "pty_orthogonalize", "pty_check_patterns",
           "pty_batch_workspace_bytes", "pty_batch_contrib", "pty_batch_apply", "pty_batch_finalize",
           "pty_accumulate",
           "pty_visit_scratch_bytes", "pty_magnitude_correct", "pty_update_object", "pty_update_probe",
           "pty_cross_power_spectrum", "pty_coarse_argmax", "pty_upsampled_idft_scratch_bytes",
           "pty_upsampled_idft", "pty_argmax_abs", "pty_adam_step", "pty_apply_correction")


def lib_path() -> Path:
    return Path(os.environ.get("PTY_LIB", str(_LIB_PATH)))


def load(require_device: bool = True):
    """Load the shared library (never builds it implicitly on a GPU box)."""
    global _lib
    with _lock:
        if _lib is None:
            p = lib_path()
            if not p.exists():
                raise NativeError(f"{p} is missing: run __graft_entry__.build() "
                                  "(python -m paper_2205_04295_b200._build)")
            _lib = _declare(C.CDLL(str(p)))
            if _lib.pty_abi_version() != 1:
                raise NativeError("libptycho_b200.so ABI mismatch")
    if require_device:
        device()
        torch().cuda.init()
    return _lib


def check(rc: int, where: str) -> None:
    if rc != 0:
        raise_for_status(int(rc), where)


def ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def dtype_code(tensor_or_dtype) -> int:
    t = torch()
    dt = getattr(tensor_or_dtype, "dtype", tensor_or_dtype)
    if dt in (t.complex64, t.float32):
        return DTYPE_C64
    if dt in (t.complex128, t.float64):
        return DTYPE_C128
    raise NativeError(f"unsupported dtype {dt}")


# --------------------------------------------------------------- workspaces --
_ws = {}


def workspace(nbytes: int, tag: str = "sweep"):
    """A cached uint8 device buffer of at least ``nbytes`` (per device, per
    stream, per tag: calls on different streams never share scratch)."""
    t = torch()
    dev = device()
    key = (dev.index, t.cuda.current_stream(dev).cuda_stream, tag)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = t.empty(max(int(nbytes), 1), dtype=t.uint8, device=dev)
        _ws[key] = buf
    return buf


# ------------------------------------------------------------------ wrappers --

def fft2(x, inverse: bool, centered: bool) -> None:
    """In-place batched 2D DFT of a contiguous (..., W, W) complex CUDA tensor."""
    lib = load()
    w = x.shape[-1]
    if x.shape[-2] != w or w not in WINDOWS or not x.is_contiguous():
        raise NativeError(f"fft2 needs contiguous square power-of-two fields, got {tuple(x.shape)}")
    batch = x.numel() // (w * w)
    check(lib.pty_fft2(ptr(x), dtype_code(x), w, batch, int(inverse), int(centered), stream_ptr()),
          "pty_fft2")


def check_patterns(patterns, status) -> None:
    lib = load()
    check(lib.pty_check_patterns(ptr(patterns), dtype_code(patterns), patterns.numel(),
                                 ptr(status), stream_ptr()), "pty_check_patterns")


def init_probes(probes, patterns, noise, window: int, modes: int) -> None:
    lib = load()
    ws = workspace(modes * window * window * 16, "init")
    check(lib.pty_init_probes(ptr(probes), dtype_code(probes), ptr(patterns), patterns.shape[0],
                              ptr(noise), window, modes, ptr(ws), ws.numel(), stream_ptr()),
          "pty_init_probes")


def orthogonalize(probes) -> None:
    lib = load()
    m, w = probes.shape[0], probes.shape[-1]
    check(lib.pty_orthogonalize(ptr(probes), dtype_code(probes), w, m, stream_ptr()),
          "pty_orthogonalize")


def sweep(args: PtySweepArgs) -> None:
    lib = load()
    check(lib.pty_sweep(C.byref(args), stream_ptr()), "pty_sweep")


def sweep_subpixel(args: PtySweepArgs) -> None:
    lib = load()
    check(lib.pty_sweep_subpixel(C.byref(args), stream_ptr()), "pty_sweep_subpixel")


def sweep_workspace_bytes(dtype: int, window: int, modes: int, n: int, slots: int) -> int:
    lib = load(require_device=False)
    b = lib.pty_sweep_workspace_bytes(dtype, window, modes, n, slots)
    if b < 0:
        raise NativeError("unsupported sweep geometry")
    return int(b)


def register_batch(work, window: int, n: int, weighting: int, kappa: int, dy, dx, peak, ok,
                   ref_real=None, mov_real=None, pairs_c64=None) -> None:
    """pty_register_batch; ``pairs_c64`` (complex64 [n][2][W][W]) are widened to
    the complex128 ``work`` while loading."""
    lib = load()
    sb = int(lib.pty_register_scratch_bytes(window, n, kappa))
    if sb < 0:
        raise NativeError("unsupported registration geometry")
    ws = workspace(sb, "register")
    real = 2 if pairs_c64 is not None else int(ref_real is not None)
    if pairs_c64 is not None:
        ref_real = pairs_c64
    check(lib.pty_register_batch(ptr(work), ptr(ref_real), ptr(mov_real), real,
                                 dtype_code(work), window, n, weighting, kappa,
                                 ptr(dy), ptr(dx), ptr(peak), ptr(ok), ptr(ws), ws.numel(),
                                 stream_ptr()), "pty_register_batch")


def adam_apply(positions, buffers, gx, gy, ok, config, bounds, index=None) -> None:
    lib = load()
    n = gx.shape[0]
    xmin, ymin, xmax, ymax = (float(b) for b in bounds)
    check(lib.pty_adam_apply(ptr(positions), ptr(buffers.m), ptr(buffers.v), ptr(buffers.t),
                             ptr(gx), ptr(gy), ptr(ok), ptr(index), n,
                             float(config.step_size), float(config.beta1), float(config.beta2),
                             float(config.eps_adam), float(config.max_correction),
                             xmin, ymin, xmax, ymax, stream_ptr()), "pty_adam_apply")


def barrier_bench(iters: int = 10000, ctas: int = 0) -> float:
    """ns per software grid barrier (sweep kernel geometry)."""
    out = C.c_double()
    check(load().pty_barrier_bench(iters, ctas, C.byref(out)), "pty_barrier_bench")
    return out.value


def timeline():
    """Debug stamps of the last sweep run with PTY_TIMELINE set: (steps, 9, grid) ns
    (0 step start, 2k-1 end of phase k, 2k barrier exit after phase k)."""
    import numpy as np
    lib = load(require_device=False)
    g = C.c_int32()
    n = lib.pty_timeline(None, 0, C.byref(g))
    buf = np.zeros(n, dtype=np.uint64)
    lib.pty_timeline(buf.ctypes.data, n, C.byref(g))
    return buf.reshape(-1, 9, g.value) if n else buf


def launch_count() -> int:
    """Kernels launched by libptycho_b200.so so far in this process."""
    return int(load(require_device=False).pty_launch_count())


def batch_workspace_bytes(dtype: int, window: int, modes: int, b: int, h: int, wc: int) -> int:
    b_ = load(require_device=False).pty_batch_workspace_bytes(dtype, window, modes, b, h, wc)
    if b_ < 0:
        raise NativeError("unsupported batch geometry")
    return int(b_)


def batch_contrib(args: PtyBatchArgs) -> None:
    check(load().pty_batch_contrib(C.byref(args), stream_ptr()), "pty_batch_contrib")


def batch_apply(args: PtyBatchArgs) -> None:
    check(load().pty_batch_apply(C.byref(args), stream_ptr()), "pty_batch_apply")


def accumulate(dst, src) -> None:
    """dst += src (contiguous real CUDA tensors of one dtype, same size)."""
    if dst.numel() != src.numel() or not dst.is_contiguous() or not src.is_contiguous():
        raise NativeError("accumulate needs two contiguous tensors of one size")
    check(load().pty_accumulate(ptr(dst), ptr(src), dst.numel(), dtype_code(dst), stream_ptr()),
          "pty_accumulate")


def batch_finalize(err_part, n_visits: int, window: int, err_out) -> None:
    check(load().pty_batch_finalize(ptr(err_part), n_visits, window, ptr(err_out), stream_ptr()),
          "pty_batch_finalize")


def device_info():
    lib = load()
    vals = [C.c_int32() for _ in range(4)]
    check(lib.pty_device_info(*[C.byref(v) for v in vals]), "pty_device_info")
    return tuple(v.value for v in vals)


# ----------------------------------------------- per-visit / per-pair calls --

def _visit_scratch(dtype: int, window: int, modes: int):
    b = int(load(require_device=False).pty_visit_scratch_bytes(dtype, window, modes))
    if b < 0:
        raise NativeError("unsupported visit geometry")
    return workspace(b, "visit")


def magnitude_correct(probes, o_j, intensity, eps_rel, corrected, psi_det, status) -> None:
    """pty_magnitude_correct on device tensors: probes/corrected/psi_det (M, W, W)."""
    lib = load()
    m, w = probes.shape[0], probes.shape[-1]
    d = dtype_code(probes)
    ws = _visit_scratch(d, w, m)
    check(lib.pty_magnitude_correct(d, w, m, ptr(probes), ptr(o_j), ptr(intensity), float(eps_rel),
                                    ptr(corrected), ptr(psi_det), ptr(status), ptr(ws), ws.numel(),
                                    stream_ptr()), "pty_magnitude_correct")


def update_object(o_j, probes, corrected, alpha, gamma, eps_rel, out, status) -> None:
    lib = load()
    m, w = probes.shape[0], probes.shape[-1]
    d = dtype_code(probes)
    ws = _visit_scratch(d, w, m)
    check(lib.pty_update_object(d, w, m, ptr(o_j), ptr(probes), ptr(corrected), float(alpha), float(gamma),
                                float(eps_rel), ptr(out), ptr(status), ptr(ws), ws.numel(), stream_ptr()),
          "pty_update_object")


def update_probe(probe, o_j, corrected, alpha, beta, eps_rel, out, status) -> None:
    lib = load()
    w = probe.shape[-1]
    d = dtype_code(probe)
    ws = _visit_scratch(d, w, 1)
    check(lib.pty_update_probe(d, w, ptr(probe), ptr(o_j), ptr(corrected), float(alpha), float(beta),
                               float(eps_rel), ptr(out), ptr(status), ptr(ws), ws.numel(), stream_ptr()),
          "pty_update_probe")


def cross_power_spectrum(work, window: int, n: int, weighting: int, xps, ok,
                         ref_real=None, mov_real=None) -> None:
    lib = load()
    sb = int(lib.pty_register_scratch_bytes(window, n, 1))
    ws = workspace(sb, "register")
    real = ref_real is not None
    check(lib.pty_cross_power_spectrum(ptr(work), ptr(ref_real), ptr(mov_real), int(real), dtype_code(work),
                                       window, n, weighting, ptr(xps), ptr(ok), ptr(ws), ws.numel(),
                                       stream_ptr()), "pty_cross_power_spectrum")


def coarse_argmax(corr, dy, dx, peak) -> None:
    lib = load()
    w = corr.shape[-1]
    n = corr.numel() // (w * w)
    check(lib.pty_coarse_argmax(ptr(corr), dtype_code(corr), w, n, ptr(dy), ptr(dx), ptr(peak), stream_ptr()),
          "pty_coarse_argmax")


def upsampled_idft(xps, rows, cols, out) -> None:
    lib = load()
    w = xps.shape[-1]
    d = dtype_code(xps)
    nr, nc = rows.numel(), cols.numel()
    sb = int(lib.pty_upsampled_idft_scratch_bytes(d, w, nr))
    ws = workspace(sb, "updft")
    check(lib.pty_upsampled_idft(ptr(xps), d, w, ptr(rows), nr, ptr(cols), nc, ptr(out), ptr(ws), ws.numel(),
                                 stream_ptr()), "pty_upsampled_idft")


def argmax_abs(x, idx, val) -> None:
    check(load().pty_argmax_abs(ptr(x), dtype_code(x), x.numel(), ptr(idx), ptr(val), stream_ptr()),
          "pty_argmax_abs")


def adam_step(buffers, j: int, gx: float, gy: float, config, delta) -> None:
    check(load().pty_adam_step(ptr(buffers.m), ptr(buffers.v), ptr(buffers.t), int(j), float(gx), float(gy),
                               float(config.step_size), float(config.beta1), float(config.beta2),
                               float(config.eps_adam), float(config.max_correction), ptr(delta), stream_ptr()),
          "pty_adam_step")


def apply_correction(positions, j: int, dx: float, dy: float, bounds, inside) -> None:
    xmin, ymin, xmax, ymax = (float(b) for b in bounds)
    check(load().pty_apply_correction(ptr(positions), int(j), float(dx), float(dy), xmin, ymin, xmax, ymax,
                                      ptr(inside), stream_ptr()), "pty_apply_correction")
