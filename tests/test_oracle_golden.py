"""Pins the CPU oracle (oracle/fftconv_oracle.c) before it is trusted as the
checker for the GPU path:

* against golden vectors produced by the REFERENCE itself
  (tests/golden/reference_golden.npz, made by tests/golden/make_golden.py
  from oracle/_ref = the reference compiled from its own headers);
* against the reference's known-answer tests (fft_test.cpp,
  conv_direct_test.cpp, acceptance criteria 4 and 7) restated here.
CPU only.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import rng

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def _cases(g):
    i = 0
    while f"c{i}_cfg" in g.files:
        yield i, tuple(int(v) for v in g[f"c{i}_cfg"])
        i += 1


def test_oracle_fft_path_matches_reference_goldens(golden):
    n_checked = 0
    for i, (k, n, f, fo, S, seed) in _cases(golden):
        for tag, dt, tol in (("f64", np.float64, 1e-14), ("f32", np.float32, 1e-6)):
            if f"c{i}_x_{tag}" not in golden.files:
                continue
            x, w, gy = golden[f"c{i}_x_{tag}"], golden[f"c{i}_w_{tag}"], golden[f"c{i}_gy_{tag}"]
            assert x.dtype == dt
            got = (oracle.forward_fft(x, w), oracle.grad_input_fft(gy, w), oracle.grad_weight_fft(gy, x))
            ref = (golden[f"c{i}_y_fft_{tag}"], golden[f"c{i}_gx_fft_{tag}"], golden[f"c{i}_gw_fft_{tag}"])
            for g_, r_ in zip(got, ref):
                assert g_.shape == r_.shape
                assert oracle.max_rel_error(g_, r_) <= tol, (i, tag)
            n_checked += 1
    assert n_checked >= 20


def test_oracle_direct_matches_reference_goldens(golden):
    for i, (k, n, f, fo, S, seed) in _cases(golden):
        if f"c{i}_y_direct_f64" not in golden.files:
            continue
        x, w, gy = golden[f"c{i}_x_f64"], golden[f"c{i}_w_f64"], golden[f"c{i}_gy_f64"]
        assert oracle.max_rel_error(oracle.forward_direct(x, w), golden[f"c{i}_y_direct_f64"]) < 1e-14
        assert oracle.max_rel_error(oracle.grad_input_direct(gy, w), golden[f"c{i}_gx_direct_f64"]) < 1e-14
        assert oracle.max_rel_error(oracle.grad_weight_direct(gy, x), golden[f"c{i}_gw_direct_f64"]) < 1e-14


def test_reference_fft_vs_direct_f64_in_goldens(golden):
    """acceptance criterion 1 (f64 1e-10) holds for the golden cases."""
    for i, _ in _cases(golden):
        if f"c{i}_y_direct_f64" not in golden.files:
            continue
        for a, b in (("y_fft_f64", "y_direct_f64"), ("gx_fft_f64", "gx_direct_f64"), ("gw_fft_f64", "gw_direct_f64")):
            assert oracle.max_rel_error(golden[f"c{i}_{a}"], golden[f"c{i}_{b}"]) < 1e-10


def test_reference_counters_in_goldens(golden):
    """The reference accumulates counters over fprop + bprop + accGrad; the
    B200 path reproduces the same analytic formula (conv_fft.hpp:108-204)."""
    for i, (k, n, f, fo, S, seed) in _cases(golden):
        m = 1
        while m < n:
            m <<= 1
        bins = m * (m // 2 + 1)
        exp = (S * f + fo * f + S * fo + fo * f + S * f + S * fo, S * fo + S * f + fo * f, 3 * bins * fo * f * S)
        assert tuple(int(v) for v in golden[f"c{i}_counters_f32"]) == exp


def test_plane_transforms_match_reference(golden):
    for key in golden.files:
        if not key.startswith("r2c_") or not key.endswith("_in"):
            continue
        m = int(key.split("_")[1][1:])
        src = golden[key]
        half = golden[key.replace("_in", "_out")]
        got = oracle.r2c_plane(src, m)
        assert np.abs(got - (half[..., 0] + 1j * half[..., 1])).max() <= 1e-13 * max(1.0, np.abs(half).max())
        back = oracle.c2r_plane(got, m, src.shape[0], src.shape[1])
        assert np.abs(back - golden[key.replace("r2c_", "c2r_").replace("_in", "_out")]).max() < 1e-13
        # the survey's restatement: reference half spectrum == numpy rfft2(s=(m, m))
        assert np.abs(got - np.fft.rfft2(src, s=(m, m))).max() < 1e-12 * max(1.0, np.abs(got).max())


def test_rng_known_answers(golden):
    """rng.hpp:32-37; SURVEY.md 8(c) known answers."""
    ref = golden["uniform_at_1234_1"]
    ours = np.array([oracle.uniform_at(1234, 1, i) for i in range(16)])
    assert np.array_equal(ours, ref)
    assert np.array_equal(rng.uniform_at(1234, 1, np.arange(16, dtype=np.uint64)), ref)
    assert ref[0] == 0.26450009843620648 and ref[1] == 0.50338282625821162 and ref[2] == 0.74215627549199059


def test_verify_config_draws_match_reference(golden):
    """bench.hpp:164-183 random_verify_configs(100, 2024)."""
    got = np.array(oracle.random_verify_configs(100, 2024), dtype=np.uint64)
    assert np.array_equal(got, golden["verify_configs_2024"])


# ----------------------------------------- fft_test.cpp known answers
def test_fft_impulse_and_dc():
    x = np.zeros(8, complex)
    x[0] = 1
    assert np.allclose(oracle.fft_1d(x), 1.0, atol=1e-14)
    c = np.full(16, 2.5 + 0j)
    X = oracle.fft_1d(c)
    assert abs(X[0] - 40) < 1e-12 and np.abs(X[1:]).max() < 1e-12
    assert np.allclose(oracle.fft_1d(X, inverse=True).real, 2.5, atol=1e-13)


@pytest.mark.parametrize("m", [2, 4, 8, 16, 32, 64])
def test_fft_matches_naive_dft(m):
    r = np.random.default_rng(m)
    x = r.standard_normal(m) + 1j * r.standard_normal(m)
    naive = np.array([sum(x[t] * np.exp(-2j * np.pi * u * t / m) for t in range(m)) for u in range(m)])
    got = oracle.fft_1d(x)
    assert np.abs(got - naive).max() / np.abs(naive).max() < 1e-12
    back = oracle.fft_1d(got, inverse=True)
    assert np.abs(back - x).max() / np.abs(x).max() < 1e-12
    # Parseval and linearity (acceptance criterion 7)
    assert abs(np.sum(np.abs(x) ** 2) - np.sum(np.abs(got) ** 2) / m) < 1e-10 * np.sum(np.abs(x) ** 2)
    y = r.standard_normal(m) + 1j * r.standard_normal(m)
    a, b = 0.7 - 0.3j, -1.1 + 0.25j
    assert np.abs(oracle.fft_1d(a * x + b * y) - (a * got + b * oracle.fft_1d(y))).max() < 1e-12 * np.abs(got).max() * 4


def test_2d_impulse_all_ones_and_back():
    p = np.zeros((8, 8))
    p[0, 0] = 1
    assert np.allclose(oracle.r2c_plane(p, 8), 1.0, atol=1e-14)
    back = oracle.c2r_plane(np.ones((8, 5), complex), 8, 8, 8)
    ref = np.zeros((8, 8))
    ref[0, 0] = 1
    assert np.abs(back - ref).max() < 1e-13


# ----------------------------------------- conv_direct_test.cpp known answers
def test_direct_hand_example():
    x = np.arange(1, 10, dtype=np.float64).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 2, 2))
    assert np.array_equal(oracle.forward_direct(x, w)[0, 0], np.array([[12.0, 16.0], [24.0, 28.0]]))
    assert np.array_equal(oracle.forward_fft(x, w).round(12)[0, 0], np.array([[12.0, 16.0], [24.0, 28.0]]))


def test_direct_delta_reproduces_kernel():
    w = np.array([[[[1.0, 2.0], [3.0, 4.0]]]])
    gx = oracle.grad_input_direct(np.ones((1, 1, 1, 1)), w)
    assert np.array_equal(gx, w)


def test_direct_adjoint_identity():
    """acceptance criterion 4 (1e-10 in f64)."""
    for (k, n, f, fo, S) in oracle.random_verify_configs(20, 77):
        no = n - k + 1
        x = oracle.fill_uniform((S, f, n, n), 77, 1, dtype=np.float64)
        w = oracle.fill_uniform((fo, f, k, k), 77, 2, dtype=np.float64)
        gy = oracle.fill_uniform((S, fo, no, no), 77, 3, dtype=np.float64)
        a = np.dot(oracle.forward_direct(x, w).ravel(), gy.ravel())
        b = np.dot(x.ravel(), oracle.grad_input_direct(gy, w).ravel())
        c = np.dot(w.ravel(), oracle.grad_weight_direct(gy, x).ravel())
        s = max(abs(a), abs(b), abs(c), 1e-30)
        assert abs(a - b) / s < 1e-10 and abs(a - c) / s < 1e-10


def test_direct_planes_subset_matches_full():
    x = oracle.fill_uniform((3, 4, 9, 9), 5, 1, dtype=np.float64)
    w = oracle.fill_uniform((5, 4, 3, 3), 5, 2, dtype=np.float64)
    gy = oracle.fill_uniform((3, 5, 7, 7), 5, 3, dtype=np.float64)
    ids = np.array([0, 7, 11])
    assert np.array_equal(oracle.forward_direct_planes(x, w, ids), oracle.forward_direct(x, w).reshape(15, 7, 7)[ids])
    assert np.array_equal(oracle.grad_input_direct_planes(gy, w, ids),
                          oracle.grad_input_direct(gy, w).reshape(12, 9, 9)[ids])
    assert np.array_equal(oracle.grad_weight_direct_planes(gy, x, ids),
                          oracle.grad_weight_direct(gy, x).reshape(20, 3, 3)[ids])
