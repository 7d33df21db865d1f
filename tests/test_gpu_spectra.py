"""The public packed-spectrum API (fft.hpp:105-152, :209-243) on the B200
kernels, against the reference's own fft_test.cpp cases (:122-199) and the
oracle (reference packing == numpy rfft2)."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import PlanError, SizeError
from paper_1312_5851_b200.spectra import HalfSpectrum, fft_2d_real_batch, ifft_2d_real_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16, 32, 64, 128])
def test_matches_reference_packing(dev, m):
    t = oracle.fill_uniform((2, 3, m, m), 500 + m, 1)
    s = fft_2d_real_batch(t)
    ref = np.fft.rfft2(t.astype(np.float64))  # == reference HalfSpectrum
    got = s.data.cpu().numpy()
    assert got.shape == ref.shape == (2, 3, m, m // 2 + 1)
    assert np.linalg.norm(got - ref) <= 2e-6 * max(np.linalg.norm(ref), 1e-30)


def test_impulse_and_constant(dev):
    """fft_test.cpp:129-150: impulse -> all ones; all ones -> m^2 at DC."""
    m = 16
    t = np.zeros((1, 2, m, m), np.float32)
    t[0, 0, 0, 0] = 1
    t[0, 1] = 1
    s = fft_2d_real_batch(t)
    assert np.allclose(s.data[0, 0].cpu().numpy(), 1.0, atol=1e-6)
    dc = s.data[0, 1].cpu().numpy()
    assert abs(dc[0, 0] - m * m) < 1e-3 and np.abs(dc).sum() - m * m < 1e-2


def test_full_bin_hermitian(dev):
    """fft_test.cpp:168-181: full_bin unpacks by Hermitian symmetry."""
    m = 8
    t = oracle.fill_uniform((1, 1, m, m), 9, 1)
    s = fft_2d_real_batch(t)
    full = np.fft.fft2(t[0, 0].astype(np.float64))
    for u in range(m):
        for v in range(m):
            assert abs(s.full_bin(0, 0, u, v) - full[u, v]) < 1e-4


@pytest.mark.parametrize("m", [4, 32, 128])
def test_round_trip(dev, m):
    """fft_test.cpp:184-193."""
    t = oracle.fill_uniform((2, 2, m, m), 70 + m, 1)
    back = ifft_2d_real_batch(fft_2d_real_batch(t)).cpu().numpy()
    assert oracle.max_rel_error(back, t) < 2e-6


def test_size_errors(dev):
    with pytest.raises(SizeError):
        fft_2d_real_batch(np.zeros((1, 1, 8, 8), np.float32), m=16)  # not padded to the plan
    with pytest.raises(PlanError):  # FftPlan(6): plan_error (fft.hpp:23-26)
        fft_2d_real_batch(np.zeros((1, 1, 6, 6), np.float32))
    with pytest.raises(SizeError):
        ifft_2d_real_batch(HalfSpectrum.zeros(1, 1, 8), m=16)
    with pytest.raises(SizeError):
        HalfSpectrum.zeros(0, 1, 8)


def test_parseval_and_packed_columns(dev):
    """fft_test.cpp:201-227: energy is preserved (sum |x|^2 = sum |X|^2 / m^2
    over the full spectrum, unpacked columns counted twice) and the packing
    keeps m/2 + 1 columns."""
    m = 32
    t = oracle.fill_uniform((2, 2, m, m), 11, 1)
    s = fft_2d_real_batch(t)
    assert s.packed_cols() == m // 2 + 1 and s.rows() == m and s.plane_size() == m * (m // 2 + 1)
    X = s.data.cpu().numpy().astype(np.complex128)
    w = np.full(m // 2 + 1, 2.0)
    w[0] = w[-1] = 1.0  # DC and Nyquist columns are their own mirrors
    energy = (np.abs(X) ** 2 * w).sum(axis=(2, 3)) / (m * m)
    ref = (t.astype(np.float64) ** 2).sum(axis=(2, 3))
    assert np.allclose(energy, ref, rtol=2e-6)


def test_linearity(dev):
    """fft_test.cpp:100-113: F(a x + b y) = a F(x) + b F(y)."""
    m = 16
    x = oracle.fill_uniform((1, 3, m, m), 21, 1)
    y = oracle.fill_uniform((1, 3, m, m), 22, 1)
    a, b = np.float32(0.75), np.float32(-2.5)
    lhs = fft_2d_real_batch(a * x + b * y).data.cpu().numpy()
    rhs = a * fft_2d_real_batch(x).data.cpu().numpy() + b * fft_2d_real_batch(y).data.cpu().numpy()
    assert np.linalg.norm(lhs - rhs) <= 1e-5 * np.linalg.norm(rhs)


@pytest.mark.parametrize("shape", [(3, 7, 32, 32), (1, 37, 8, 8), (2, 9, 64, 64), (1, 19, 128, 128), (4, 5, 2, 2)])
def test_many_planes_round_trip(dev, shape):
    """Plane counts off the 16-plane grouping, every FFT-size family, through
    the C-ABI batch entry points (fftconv_b200_fft_2d_real_batch / _ifft_)."""
    t = oracle.fill_uniform(shape, 31 + shape[1], 1)
    s = fft_2d_real_batch(t)
    ref = np.fft.rfft2(t.astype(np.float64))
    assert np.linalg.norm(s.data.cpu().numpy() - ref) <= 2e-6 * np.linalg.norm(ref)
    back = ifft_2d_real_batch(s).cpu().numpy()
    assert np.linalg.norm(back - t) <= 2e-6 * np.linalg.norm(t)
