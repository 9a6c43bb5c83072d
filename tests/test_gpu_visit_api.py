"""The reference's per-visit / per-pair public functions on the GPU (C ABI
pty_magnitude_correct ... pty_apply_correction, csrc/pty_visit.cu).

Restates the assertions of the reference's own tests against this package:
  /root/reference/pkg/tests/test_engine.py:98-142   (magnitude_correct, update rules)
  /root/reference/pkg/tests/test_registration.py:32-157 (cross_power_spectrum,
                                                      coarse_shift, upsampled_idft, refine_shift)
  /root/reference/pkg/tests/test_posref.py:14-133   (sensors, adam_step, apply_correction)
Deviation: fields must be power-of-two squares >= 16, so
the reference's 8x8 degenerate-input cases run at 16x16 and the 12x12 / 24x24
registration cases at 16x16 / 32x32.
"""

import numpy as np
import pytest
from scipy.ndimage import gaussian_filter

import paper_2205_04295_b200 as pk
from paper_2205_04295_b200.engine import magnitude_correct, update_object, update_probe
from paper_2205_04295_b200.errors import DataError, DegenerateInputError, ParameterError, ShapeError
from paper_2205_04295_b200.fields import CropBox, crop, subpixel_shift
from paper_2205_04295_b200.posref import (AdamBuffers, PosRefConfig, adam_step, apply_correction,
                                          sense_shift_A, sense_shift_B)
from paper_2205_04295_b200.registration import (coarse_shift, cross_power_spectrum, refine_shift, register,
                                                upsampled_idft)

pytestmark = pytest.mark.gpu

GEOM = pk.Geometry.create(8.3187e-10, 0.75, 20e-6, 32)


def scene(mode_count=1, powers=(1.0,), grid=(4, 4), step=7.0, jitter=0.0, seed=3):
    plan = pk.make_scan(grid, step, jitter, seed=seed)
    obj = pk.make_object(pk.canvas_shape_for(plan, 32), "spokes", seed=seed)
    probes = pk.make_probe(pk.ProbeSpec(mode_count, powers, "disk", 8.0), GEOM)
    ds = pk.synthesize(obj, probes, plan, GEOM)
    return obj, probes, plan, ds


def fft_c(a):
    return np.fft.fftshift(np.fft.fft2(np.fft.ifftshift(a), norm="ortho"))


def ifft_c(a):
    return np.fft.fftshift(np.fft.ifft2(np.fft.ifftshift(a), norm="ortho"))


def reference_rpie_step(o_j, probes, i_j, alpha_o, alpha_p, beta, gamma, eps_rel=1e-12):
    """Straight-line numpy visit (the reference test's own oracle, test_engine.py:37-59)."""
    psi_det = [fft_c(p * o_j) for p in probes]
    total = sum(np.abs(psi) ** 2 for psi in psi_det)
    eps = eps_rel * max(total.max(), np.finfo(float).tiny)
    corrected = [ifft_c(np.sqrt(i_j) * psi / np.sqrt(total + eps)) for psi in psi_det]
    probe_power = sum(np.abs(p) ** 2 for p in probes)
    denom_o = gamma * probe_power.max() + (1 - gamma) * probe_power
    denom_o = denom_o + eps_rel * denom_o.max()
    numer = sum((c - p * o_j) * np.conj(p) for p, c in zip(probes, corrected))
    new_o = o_j + alpha_o * numer / denom_o
    obj_power = np.abs(o_j) ** 2
    denom_p = beta * obj_power.max() + (1 - beta) * obj_power
    denom_p = denom_p + eps_rel * denom_p.max()
    new_probes = [p + alpha_p * (c - p * o_j) * np.conj(o_j) / denom_p for p, c in zip(probes, corrected)]
    return new_o, new_probes


def close(got, want, rtol=1e-12):
    """Element-wise rtol plus an absolute floor at round-off of the field's
    scale (a different FFT than pocketfft differs by ulps of the largest
    element, which is not small relative to the smallest ones)."""
    np.testing.assert_allclose(got, want, rtol=rtol, atol=1e-13 * np.max(np.abs(want)))


# ------------------------------------------------------- engine.py:104-150 ----

def test_corrected_waves_reproduce_measurement(gpu):
    obj, probes, plan, ds = scene(mode_count=2, powers=(0.8, 0.2))
    o_j = np.asarray(crop(obj, CropBox(0, 0, 32)))
    i_j = ds.patterns[0]
    corrected, psi_det = magnitude_correct(probes, o_j, i_j)
    after = sum(np.abs(fft_c(c)) ** 2 for c in corrected)
    total = sum(np.abs(p) ** 2 for p in psi_det)
    guard = total > 1e-3 * total.max()
    assert guard.any()
    np.testing.assert_allclose(after[guard], i_j[guard], rtol=1e-9)
    for p, d in zip(probes, psi_det):
        close(d, fft_c(p * o_j))


def test_magnitude_correct_rejects_negative_intensity(gpu):
    _, probes, _, ds = scene()
    bad = ds.patterns[0].copy()
    bad[0, 0] = -1.0
    with pytest.raises(DataError):
        magnitude_correct(probes, np.ones((32, 32), complex), bad)


@pytest.mark.parametrize("beta,gamma", [(1.0, 1.0), (0.3, 0.25), (0.9, 0.05)])
def test_single_visit_matches_reference_implementation(gpu, beta, gamma):
    obj, probes, plan, ds = scene(mode_count=2, powers=(0.7, 0.3))
    o_j = np.asarray(crop(obj, CropBox(2, 3, 32)))
    i_j = ds.patterns[5]
    want_o, want_p = reference_rpie_step(o_j, probes, i_j, 0.9, 0.8, beta, gamma)
    corrected, _ = magnitude_correct(probes, o_j, i_j)
    got_o = update_object(o_j, probes, corrected, 0.9, gamma)
    got_p = [update_probe(p, o_j, c, 0.8, beta) for p, c in zip(probes, corrected)]
    close(got_o, want_o)
    for g, w in zip(got_p, want_p):
        close(g, w)


def test_visit_functions_fp32_tensors(gpu):
    """torch complex64 inputs stay on the device and run the fp32 kernels."""
    import torch
    obj, probes, plan, ds = scene(mode_count=2, powers=(0.7, 0.3))
    o_j = np.asarray(crop(obj, CropBox(2, 3, 32)))
    i_j = ds.patterns[5]
    want_o, want_p = reference_rpie_step(o_j, probes, i_j, 0.9, 0.8, 0.5, 0.5)
    pt = torch.from_numpy(np.stack(probes)).to("cuda", torch.complex64)
    ot = torch.from_numpy(o_j).to("cuda", torch.complex64)
    it = torch.from_numpy(i_j).to("cuda", torch.float32)
    corrected, _ = magnitude_correct(pt, ot, it)
    got_o = update_object(ot, pt, corrected, 0.9, 0.5)
    assert got_o.dtype == torch.complex64 and got_o.is_cuda
    got_p = update_probe(pt[0], ot, corrected[0], 0.8, 0.5)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(got_o.cpu().numpy(), want_o) < 1e-6
    assert rel(got_p.cpu().numpy(), want_p[0]) < 1e-5


def test_degenerate_inputs_rejected(gpu):
    z = np.zeros((16, 16), complex)
    with pytest.raises(DegenerateInputError):
        update_object(np.ones((16, 16), complex), [z], [z], 0.9, 1.0)
    with pytest.raises(DegenerateInputError):
        update_probe(np.ones((16, 16), complex), z, z, 0.9, 1.0)


# ------------------------------------------------- registration.py:43-120 ----

def smooth_image(side, seed=0, sigma=2.0):
    rng = np.random.default_rng(seed)
    return gaussian_filter(rng.standard_normal((side, side)), sigma)


def brute_force_xcorr(ref, mov):
    n = ref.shape[0]
    out = np.zeros((n, n), complex)
    for uy in range(n):
        for ux in range(n):
            out[uy, ux] = np.sum(np.roll(ref, (-uy, -ux), axis=(0, 1)) * np.conj(mov))
    return out


def test_identical_inputs_give_centered_impulse(gpu):
    f = smooth_image(16, 1)
    xps = cross_power_spectrum(f, f, "phase")
    corr = np.abs(np.fft.fftshift(np.fft.ifft2(xps)))
    assert np.unravel_index(np.argmax(corr), corr.shape) == (8, 8)
    flat = np.sort(corr.ravel())
    assert flat[-1] > 100 * flat[-2]


def test_raw_spectrum_matches_brute_force(gpu):
    rng = np.random.default_rng(5)
    ref = rng.standard_normal((16, 16))
    mov = rng.standard_normal((16, 16))
    xps = cross_power_spectrum(ref, mov, "raw")
    fast = np.fft.ifft2(xps)
    slow = brute_force_xcorr(ref, mov)
    assert np.max(np.abs(fast - slow)) < 1e-8 * np.max(np.abs(slow))


def test_conjugate_symmetry_for_real_inputs(gpu):
    ref = smooth_image(16, 2)
    mov = smooth_image(16, 3)
    xps = cross_power_spectrum(ref, mov, "raw")
    flipped = np.conj(np.roll(xps[::-1, ::-1], (1, 1), axis=(0, 1)))
    assert np.allclose(xps, flipped, atol=1e-9 * np.abs(xps).max())


def test_cross_power_spectrum_errors(gpu):
    z = np.zeros((16, 16))
    with pytest.raises(DegenerateInputError):
        cross_power_spectrum(z, z)
    with pytest.raises(ShapeError):
        cross_power_spectrum(np.ones((16, 16)), np.ones((32, 32)))
    with pytest.raises(ParameterError):
        cross_power_spectrum(smooth_image(16), smooth_image(16), "hann")


def test_coarse_zero_shift(gpu):
    f = smooth_image(16, 4)
    est = coarse_shift(cross_power_spectrum(f, f))
    assert (est.dy, est.dx) == (0.0, 0.0)


@pytest.mark.parametrize("shift", [(5, -3), (0, 7), (-6, -6), (16, 1)])
def test_integer_roll_recovered(gpu, shift):
    f = smooth_image(32, 5)
    mov = np.roll(f, shift, axis=(0, 1))
    est = coarse_shift(cross_power_spectrum(f, mov))
    want = (-((shift[0] + 16) % 32 - 16), -((shift[1] + 16) % 32 - 16))
    assert (est.dy, est.dx) == want


def test_coarse_tie_breaks(gpu):
    est = coarse_shift(np.ones((16, 16), complex))
    assert (est.dy, est.dx) == (0.0, 0.0)
    corr = np.zeros((16, 16))
    corr[8 + 1, 8] = 1.0
    corr[8 + 5, 8] = 1.0
    est = coarse_shift(np.fft.fft2(np.fft.ifftshift(corr)))
    assert (est.dy, est.dx) == (1.0, 0.0)


def test_upsampled_idft_matches_ifft2_on_integer_grid(gpu):
    rng = np.random.default_rng(6)
    xps = rng.standard_normal((16, 16)) + 1j * rng.standard_normal((16, 16))
    full = np.fft.ifft2(xps)
    got = upsampled_idft(xps, np.array([0.0, 3.0, -2.0]), np.array([1.0, -5.0]))
    for i, r in enumerate([0, 3, -2]):
        for k, c in enumerate([1, -5]):
            assert got[i, k] == pytest.approx(full[r % 16, c % 16], abs=1e-12)


def test_refine_shift_api(gpu):
    f = smooth_image(16, 7)
    xps = cross_power_spectrum(f, f)
    coarse = coarse_shift(xps)
    assert refine_shift(xps, coarse, 1) is coarse
    for kappa in (0, -3, 1001):
        with pytest.raises(ParameterError):
            refine_shift(xps, coarse, kappa)
    ref = smooth_image(32, 9)
    mov = np.asarray(subpixel_shift(ref, 0.25, -0.75)).real
    xps = cross_power_spectrum(ref, mov, "phase")
    est = refine_shift(xps, coarse_shift(xps), 20)
    assert est.dx == pytest.approx(-0.25, abs=0.05) and est.dy == pytest.approx(0.75, abs=0.05)
    # the composed steps equal the fused batched pipeline exactly
    fused = register(ref, mov, "phase", 20)
    assert (fused.dy, fused.dx) == (est.dy, est.dx)
    assert fused.peak_value == pytest.approx(est.peak_value, rel=1e-9)


def test_refine_containment_near_coarse(gpu):
    rng = np.random.default_rng(11)
    for seed in range(20):
        ref = smooth_image(16, 100 + seed, sigma=1.0)
        mov = smooth_image(16, 200 + seed, sigma=1.0)
        xps = cross_power_spectrum(ref, mov, "phase")
        coarse = coarse_shift(xps)
        fine = refine_shift(xps, coarse, int(rng.integers(2, 60)))
        assert abs(fine.dy - coarse.dy) <= 0.75 + 1e-12
        assert abs(fine.dx - coarse.dx) <= 0.75 + 1e-12


# ------------------------------------------------------- posref.py:57-113 ----

def crop_from_object(seed=3, side=32):
    return pk.make_object((side, side), "phase-screen", seed=seed)


def test_sense_shift_a(gpu):
    o = crop_from_object()
    gx, gy, ok = sense_shift_A(o, o, kappa=100)
    assert ok and gx == 0.0 and gy == 0.0
    moved = np.asarray(subpixel_shift(o, -0.4, 0.0))
    gx, gy, ok = sense_shift_A(o, moved, kappa=100)
    assert ok and gx == pytest.approx(0.4, abs=2 / 100) and gy == pytest.approx(0.0, abs=2 / 100)
    moved = np.asarray(subpixel_shift(o, -0.3, 0.2))
    fwd = sense_shift_A(o, moved, kappa=100)
    rev = sense_shift_A(moved, o, kappa=100)
    assert fwd[0] == pytest.approx(-rev[0], abs=2 / 100) and fwd[1] == pytest.approx(-rev[1], abs=2 / 100)
    flat = np.zeros((32, 32), dtype=complex)
    assert sense_shift_A(flat, flat, kappa=100) == (0.0, 0.0, False)


def test_sense_shift_b(gpu):
    i = np.abs(crop_from_object()) ** 2
    gx, gy, ok = sense_shift_B(i, i, kappa=100)
    assert ok and gx == 0.0 and gy == 0.0
    gx, gy, ok = sense_shift_B(i, np.roll(i, 2, axis=1), kappa=10)
    assert ok and (abs(gx) > 0.5 or abs(gy) > 0.5)


def test_adam_step_behaviour(gpu):
    buf = AdamBuffers.zeros(2)
    dx, dy = adam_step(buf, 0, (0.0, 0.0), PosRefConfig())
    assert dx == 0.0 and dy == 0.0
    assert int(buf.t[0]) == 1 and int(buf.t[1]) == 0
    buf = AdamBuffers.zeros(1)
    dx, dy = adam_step(buf, 0, (1e-3, -1e-3), PosRefConfig(step_size=0.5))
    assert dx == pytest.approx(0.5, rel=1e-4) and dy == pytest.approx(-0.5, rel=1e-4)
    buf = AdamBuffers.zeros(1)
    for _ in range(50):
        dx, dy = adam_step(buf, 0, (0.01, 0.01), PosRefConfig(step_size=0.2))
    assert dx == pytest.approx(0.2, rel=1e-3) and abs(dx) <= 0.2 + 1e-12
    buf = AdamBuffers.zeros(1)
    for k in range(40):
        dx, _ = adam_step(buf, 0, (0.05 if k % 2 == 0 else -0.05, 0.0), PosRefConfig(step_size=0.5))
    assert abs(dx) < 0.15
    buf = AdamBuffers.zeros(1)
    assert adam_step(buf, 0, (1.0, 1.0), PosRefConfig(step_size=5.0, max_correction=0.7)) == (0.7, 0.7)
    buf = AdamBuffers.zeros(3)
    for _ in range(5):
        adam_step(buf, 0, (0.1, 0.0), PosRefConfig())
    m, v, t = buf.numpy()
    assert t[0] == 5 and np.all(m[1:] == 0) and np.all(v[1:] == 0) and np.all(t[1:] == 0)


def test_adam_moment_recurrences_match_reference(gpu):
    cfg = PosRefConfig(step_size=0.3, beta1=0.8, beta2=0.95, max_correction=10)
    buf = AdamBuffers.zeros(1)
    rng = np.random.default_rng(1)
    m = np.zeros(2)
    v = np.zeros(2)
    for t in range(1, 8):
        g = rng.uniform(-1, 1, 2)
        m = 0.8 * m + 0.2 * g
        v = 0.95 * v + 0.05 * g * g
        want = 0.3 * (m / (1 - 0.8 ** t)) / (np.sqrt(v / (1 - 0.95 ** t)) + cfg.eps_adam)
        np.testing.assert_allclose(adam_step(buf, 0, tuple(g), cfg), want, rtol=1e-12)


def test_apply_correction(gpu):
    import torch
    pos = np.array([[5.0, 5.0]])
    assert apply_correction(pos, 0, (0.25, -0.5), (0.0, 0.0, 10.0, 10.0))
    np.testing.assert_allclose(pos[0], [5.25, 4.5])
    pos = np.array([[9.9, 0.1]])
    assert not apply_correction(pos, 0, (0.5, -0.5), (0.0, 0.0, 10.0, 10.0))
    np.testing.assert_allclose(pos[0], [10.0, 0.0])
    dev = torch.tensor([[1.0, 2.0], [9.9, 0.1]], dtype=torch.float64, device="cuda")
    assert not apply_correction(dev, 1, (0.5, -0.5), (0.0, 0.0, 10.0, 10.0))
    np.testing.assert_allclose(dev.cpu().numpy(), [[1.0, 2.0], [10.0, 0.0]])
