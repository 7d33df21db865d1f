"""Unit parity of the individual B200 kernels (K1 r2c, K4 c2r, K3 per-bin
complex GEMM) against the oracle / numpy.  These localise a failure before
the operator-level tests in test_gpu_parity.py."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _rel(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("m,src", [(1, 1), (2, 2), (4, 3), (8, 5), (8, 8), (16, 9), (16, 16),
                                   (32, 7), (32, 26), (32, 32), (64, 11), (64, 54), (64, 64)])
def test_r2c_matches_dft(dev, m, src):
    import torch

    from paper_1312_5851_b200 import kernels

    P = 37
    x = oracle.fill_uniform((P, src, src), 7 + m + src, 1)
    got = kernels.r2c(torch.from_numpy(x).to(dev), m).cpu().numpy()
    pad = np.zeros((P, m, m))
    pad[:, :src, :src] = x
    full = np.fft.fft2(pad)
    ref = full[:, : m // 2 + 1, :]  # half over rows u, all columns v
    assert got.shape == ref.shape
    assert _rel(got, ref) < 2e-6


@pytest.mark.parametrize("m", [1, 2, 4, 8, 16, 32, 64])
def test_r2c_impulse_is_all_ones(dev, m):
    """fft_test.cpp:129-139: an impulse at the origin has an all-ones spectrum."""
    import torch

    from paper_1312_5851_b200 import kernels

    x = np.zeros((1, m, m), dtype=np.float32)
    x[0, 0, 0] = 1
    got = kernels.r2c(torch.from_numpy(x).to(dev), m).cpu().numpy()
    assert np.allclose(got, 1.0, atol=1e-6)


@pytest.mark.parametrize("m,crop", [(1, 1), (2, 2), (4, 3), (8, 8), (16, 11), (32, 26), (32, 32),
                                    (32, 7), (64, 54), (64, 64), (64, 11)])
def test_c2r_matches_numpy(dev, m, crop):
    import torch

    from paper_1312_5851_b200 import kernels

    P = 19
    rng = np.random.default_rng(m * 100 + crop)
    H = rng.standard_normal((P, m // 2 + 1, m)) + 1j * rng.standard_normal((P, m // 2 + 1, m))
    got = kernels.c2r(torch.from_numpy(H.astype(np.complex64)).to(dev), crop).cpu().numpy()
    ref = np.fft.irfft(np.fft.ifft(H, axis=2), n=m, axis=1)[:, :crop, :crop]
    assert _rel(got, ref) < 2e-6


@pytest.mark.parametrize("m,src", [(16, 16), (32, 26), (64, 64)])
def test_r2c_c2r_round_trip(dev, m, src):
    """fft_test.cpp:184-193 round trip, through the B200 kernels."""
    import torch

    from paper_1312_5851_b200 import kernels

    x = oracle.fill_uniform((9, src, src), 99, 1)
    spec = kernels.r2c(torch.from_numpy(x).to(dev), m)
    back = kernels.c2r(spec, src).cpu().numpy()
    assert oracle.max_rel_error(back, x) < 2e-6


@pytest.mark.parametrize("bins,M,N,K", [(3, 8, 16, 16), (5, 128, 96, 96), (2, 96, 96, 128),
                                        (4, 5, 3, 7), (2, 200, 40, 20), (3, 128, 256, 64),
                                        (2, 130, 130, 33), (2, 64, 48, 48), (3, 40, 100, 80)])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_cgemm_bins(dev, gemm_kind, bins, M, N, K, mode):
    import torch

    from paper_1312_5851_b200 import kernels

    g = torch.Generator().manual_seed(bins * 1000 + M + N + K + mode)
    a = torch.complex(torch.randn(bins, M, K, generator=g), torch.randn(bins, M, K, generator=g))
    b = torch.complex(torch.randn(bins, N, K, generator=g), torch.randn(bins, N, K, generator=g))
    got = kernels.cgemm(a.to(dev), b.to(dev), mode).cpu().to(torch.complex128)
    A, B = a.to(torch.complex128), b.to(torch.complex128)
    if mode == 0:
        ref = torch.einsum("tmk,tnk->tnm", A, B.conj())
    elif mode == 1:
        ref = torch.einsum("tmk,tnk->tnm", A, B)
    else:
        ref = torch.einsum("tmk,tnk->tnm", A.conj(), B)
    err = float((got - ref).abs().norm() / ref.abs().norm())
    # 3xTF32 and fp16x3 hold fp32-level accuracy; plain TF32 would sit near 3e-4.
    assert err < 5e-6, err


@pytest.mark.parametrize("scale_a,scale_b", [(2.0 ** -60, 2.0 ** 50), (1e-30, 1e-8), (1e20, 1e15), (0.0, 1.0)])
def test_cgemm_operand_scaling(dev, gemm_kind, scale_a, scale_b):
    """fp16x3 rescales each operand by a power of two from its max magnitude:
    results far outside the fp16 range (and all-zero operands) stay exact to
    fp32 level."""
    import torch

    from paper_1312_5851_b200 import kernels

    g = torch.Generator().manual_seed(5)
    a = torch.complex(torch.randn(3, 70, 40, generator=g), torch.randn(3, 70, 40, generator=g)) * scale_a
    b = torch.complex(torch.randn(3, 50, 40, generator=g), torch.randn(3, 50, 40, generator=g)) * scale_b
    got = kernels.cgemm(a.to(dev), b.to(dev), 0).cpu().to(torch.complex128)
    ref = torch.einsum("tmk,tnk->tnm", a.to(torch.complex128), b.to(torch.complex128).conj())
    assert torch.isfinite(got.real).all() and torch.isfinite(got.imag).all()
    if scale_a == 0.0:
        assert float(got.abs().max()) == 0.0
        return
    err = float((got - ref).abs().norm() / ref.abs().norm())
    assert err < 5e-6, err


def test_cgemm_wide_dynamic_range_rows(dev, gemm_kind):
    """Rows spanning 2^20 in magnitude within one operand: each output row
    keeps its own relative accuracy (fp16x3 scales by the operand maximum;
    components below ~2^-24 of it reach fp16's subnormal floor and keep only
    an absolute error of ~2^-38 of the maximum)."""
    import torch

    from paper_1312_5851_b200 import kernels

    g = torch.Generator().manual_seed(6)
    rows = (2.0 ** torch.linspace(-10, 10, 64)).reshape(1, 64, 1)
    a = torch.complex(torch.randn(2, 64, 32, generator=g), torch.randn(2, 64, 32, generator=g)) * rows
    b = torch.complex(torch.randn(2, 32, 32, generator=g), torch.randn(2, 32, 32, generator=g))
    got = kernels.cgemm(a.to(dev), b.to(dev), 0).cpu().to(torch.complex128)
    ref = torch.einsum("tmk,tnk->tnm", a.to(torch.complex128), b.to(torch.complex128).conj())
    # per output row m: error relative to that row's norm
    num = (got - ref).abs().pow(2).sum(dim=(0, 1)).sqrt()
    den = ref.abs().pow(2).sum(dim=(0, 1)).sqrt()
    rel = (num / den).max().item()
    assert rel < 2e-5, rel
