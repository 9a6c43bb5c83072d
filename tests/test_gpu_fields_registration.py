"""Property tests of the reference's fields/registration suites
(/root/reference/pkg/tests/test_fields.py:58-175, test_registration.py:32-195)
run on this package's GPU implementations (propagate, crop/paste, subpixel
shift, register).  Windows are powers of two here."""

import numpy as np
import pytest
from scipy.ndimage import gaussian_filter

import paper_2205_04295_b200 as pk
from paper_2205_04295_b200 import errors
from paper_2205_04295_b200.fields import CropBox, crop, paste_add, paste_add_inplace, subpixel_shift

pytestmark = pytest.mark.gpu


def host(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def random_field(n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))


def smooth_image(n, seed, sigma=2.0):
    return gaussian_filter(np.random.default_rng(seed).standard_normal((n, n)), sigma)


# --------------------------------------------------------------- fields ----
def test_centered_impulse_becomes_flat(gpu):
    f = np.zeros((16, 16), complex)
    f[8, 8] = 1.0
    out = host(pk.propagate(f))
    np.testing.assert_allclose(np.abs(out), np.full((16, 16), 1 / 16), atol=1e-14)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_round_trip_and_parseval(gpu, seed):
    f = random_field(32, seed)
    back = host(pk.propagate(pk.propagate(f), "backward"))
    assert np.max(np.abs(back - f)) < 1e-12
    assert np.sum(np.abs(host(pk.propagate(f))) ** 2) == pytest.approx(np.sum(np.abs(f) ** 2), rel=1e-12)


def test_propagate_rejects(gpu):
    with pytest.raises(errors.ShapeError):
        pk.propagate(np.ones((8, 16), complex))
    with pytest.raises((errors.ParameterError, ValueError)):
        pk.propagate(np.ones((8, 8), complex), "sideways")


def test_crop_and_paste_properties(gpu):
    out = crop(np.ones((20, 20), complex), CropBox(3, 5, 8))
    assert out.shape == (8, 8) and np.all(out == 1.0)
    canvas = np.arange(100, dtype=complex).reshape(10, 10)
    assert np.array_equal(crop(canvas, CropBox(0, 0, 4)), canvas[:4, :4])
    with pytest.raises(errors.BoundsError):
        crop(np.ones((10, 10), complex), CropBox(5, 5, 8))
    z = np.zeros((10, 10), complex)
    c = crop(z, CropBox(0, 0, 4))
    c += 1
    assert np.all(z == 0)
    canvas = random_field(16, 4)
    d1, d2 = random_field(4, 5), random_field(4, 6)
    b1, b2 = CropBox(0, 0, 4), CropBox(8, 8, 4)
    assert np.array_equal(paste_add(paste_add(canvas, b1, d1), b2, d2),
                          paste_add(paste_add(canvas, b2, d2), b1, d1))
    box = CropBox(4, 4, 4)
    out = paste_add(canvas, box, random_field(4, 10))
    mask = np.ones((16, 16), bool)
    mask[4:8, 4:8] = False
    assert np.array_equal(out[mask], canvas[mask])
    with pytest.raises(errors.ShapeError):
        paste_add_inplace(np.zeros((10, 10), complex), CropBox(0, 0, 4), np.zeros((5, 5), complex))


def test_subpixel_shift_properties(gpu):
    f = random_field(16, 1)
    assert np.max(np.abs(host(subpixel_shift(f, 0, 0)) - f)) < 1e-12
    np.testing.assert_allclose(host(subpixel_shift(f, 3, -2)), np.roll(f, (-2, 3), axis=(0, 1)), atol=1e-12)
    half = host(subpixel_shift(host(subpixel_shift(f, 0.5, 0.25)), 0.5, 0.25))
    np.testing.assert_allclose(half, host(subpixel_shift(f, 1.0, 0.5)), atol=1e-12)
    with pytest.raises(errors.ShapeError):
        subpixel_shift(f, 8.0, 0.0)


# --------------------------------------------------------- registration ----
def test_self_registration_and_integer_rolls(gpu):
    f = smooth_image(32, 12)
    est = pk.register(f, f, "phase", 10)
    assert (est.dy, est.dx) == (0.0, 0.0)
    rng = np.random.default_rng(14)
    ref = rng.standard_normal((16, 16))
    for shift in [(2, 3), (-4, 1), (0, -5)]:
        mov = np.roll(ref, shift, axis=(0, 1))
        est = pk.register(ref, mov, "raw", 1)
        assert (est.dy, est.dx) == (-shift[0], -shift[1])


def test_known_subpixel_shift_and_antisymmetry(gpu):
    ref = smooth_image(32, 9)
    mov = host(subpixel_shift(ref, 0.25, -0.75)).real
    est = pk.register(ref, mov, "phase", 20)
    assert est.dx == pytest.approx(-0.25, abs=0.05)
    assert est.dy == pytest.approx(0.75, abs=0.05)
    ref = smooth_image(32, 13)
    mov = host(subpixel_shift(ref, 1.2, -0.6)).real
    ab = pk.register(ref, mov, "phase", 25)
    ba = pk.register(mov, ref, "phase", 25)
    assert ab.dy == pytest.approx(-ba.dy, abs=2 / 25)
    assert ab.dx == pytest.approx(-ba.dx, abs=2 / 25)


def test_monotone_improvement_with_upsampling(gpu):
    errs = {1: [], 20: []}
    for seed in range(30):
        ref = smooth_image(32, 300 + seed)
        dx, dy = np.random.default_rng(400 + seed).uniform(-3, 3, 2)
        mov = host(subpixel_shift(ref, dx, dy)).real
        for kappa in (1, 20):
            est = pk.register(ref, mov, "phase", kappa)
            errs[kappa].append(max(abs(est.dx + dx), abs(est.dy + dy)))
    assert max(errs[20]) <= max(errs[1]) + 1 / 20


def test_registration_rejects(gpu):
    z = np.zeros((16, 16))
    with pytest.raises(errors.DegenerateInputError):
        pk.register(z, z)
    with pytest.raises(errors.ShapeError):
        pk.register(np.ones((16, 16)), np.ones((8, 8)))
    with pytest.raises(errors.ParameterError):
        pk.register(np.ones((16, 16)), np.ones((16, 16)), weighting="tukey")
    for kappa in (0, -3, 1001):
        with pytest.raises(errors.ParameterError):
            pk.register(smooth_image(16, 8), smooth_image(16, 8), "phase", kappa)
