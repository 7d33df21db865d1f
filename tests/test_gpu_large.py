"""FFT size m = 128 (image edges 65..128; BASELINE configs[4]'s first layer,
n = 128): the two-pass K1 / K4 kernels of fft_large.cuh in isolation against
numpy, and the three operators against the fp64 direct oracle at the
reference's rel-L2 1e-4 bar (acceptance_test.cpp:47), including operand-row
chunking of the scratch (forced small by FFTCONV_B200_LSCRATCH_MB)."""
import os

import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig, SizeError

pytestmark = pytest.mark.gpu


def _rel(got, ref):
    return float(np.linalg.norm(np.asarray(got) - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.mark.parametrize("src", [11, 65, 118, 128])
def test_r2c128_matches_dft(dev, src):
    import torch

    from paper_1312_5851_b200 import kernels

    P = 5
    x = oracle.fill_uniform((P, src, src), 300 + src, 1)
    got = kernels.r2c(torch.from_numpy(x).to(dev), 128).cpu().numpy()
    pad = np.zeros((P, 128, 128))
    pad[:, :src, :src] = x
    ref = np.fft.fft2(pad)[:, :65, :]
    assert got.shape == ref.shape
    assert _rel(got, ref) < 2e-6


def test_r2c128_impulse_is_all_ones(dev):
    import torch

    from paper_1312_5851_b200 import kernels

    x = np.zeros((1, 128, 128), dtype=np.float32)
    x[0, 0, 0] = 1
    assert np.allclose(kernels.r2c(torch.from_numpy(x).to(dev), 128).cpu().numpy(), 1.0, atol=1e-6)


@pytest.mark.parametrize("crop", [11, 65, 118, 128])
def test_c2r128_matches_numpy(dev, crop):
    import torch

    from paper_1312_5851_b200 import kernels

    P = 7
    rng = np.random.default_rng(crop)
    H = rng.standard_normal((P, 65, 128)) + 1j * rng.standard_normal((P, 65, 128))
    got = kernels.c2r(torch.from_numpy(H.astype(np.complex64)).to(dev), crop).cpu().numpy()
    ref = np.fft.irfft(np.fft.ifft(H, axis=2), n=128, axis=1)[:, :crop, :crop]
    assert _rel(got, ref) < 2e-6


@pytest.mark.parametrize("src", [118, 128])
def test_r2c128_staged_path_matches_dft(dev, monkeypatch, src):
    """FFTCONV_B200_LBULK=0: even planes through the staged K1a / K4b instead
    of the bulk-copy ones; same spectra and crops."""
    import torch

    from paper_1312_5851_b200 import kernels

    monkeypatch.setenv("FFTCONV_B200_LBULK", "0")
    P = 3
    x = oracle.fill_uniform((P, src, src), 310 + src, 1)
    got = kernels.r2c(torch.from_numpy(x).to(dev), 128).cpu().numpy()
    pad = np.zeros((P, 128, 128))
    pad[:, :src, :src] = x
    assert _rel(got, np.fft.fft2(pad)[:, :65, :]) < 2e-6
    rng = np.random.default_rng(src)
    H = rng.standard_normal((P, 65, 128)) + 1j * rng.standard_normal((P, 65, 128))
    back = kernels.c2r(torch.from_numpy(H.astype(np.complex64)).to(dev), src).cpu().numpy()
    assert _rel(back, np.fft.irfft(np.fft.ifft(H, axis=2), n=128, axis=1)[:, :src, :src]) < 2e-6


def test_r2c128_unaligned_planes_take_staged_path(dev):
    """Planes 4 B off 16-B alignment cannot be bulk-copied: the host picks the
    staged K1a for them (same result)."""
    import torch

    from paper_1312_5851_b200 import kernels

    P, src = 3, 118
    x = oracle.fill_uniform((P, src, src), 320, 1)
    flat = torch.zeros(P * src * src + 4, dtype=torch.float32, device=dev)
    view = flat[1:1 + P * src * src].view(P, src, src)
    view.copy_(torch.from_numpy(x))
    assert view.data_ptr() % 16 != 0 and view.is_contiguous()
    got = kernels.r2c(view, 128).cpu().numpy()
    pad = np.zeros((P, 128, 128))
    pad[:, :src, :src] = x
    assert _rel(got, np.fft.fft2(pad)[:, :65, :]) < 2e-6


def test_r2c_c2r128_round_trip(dev):
    import torch

    from paper_1312_5851_b200 import kernels

    x = oracle.fill_uniform((3, 100, 100), 5, 1)
    back = kernels.c2r(kernels.r2c(torch.from_numpy(x).to(dev), 128), 100).cpu().numpy()
    assert oracle.max_rel_error(back, x) < 2e-6


def _inputs(cfg, seed):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    return (oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT),
            oracle.fill_uniform((fo, f, k, k), seed, oracle.ROLE_WEIGHTS),
            oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT))


def _check_ops(cfg, seed, dev, ws=None):
    import torch

    x, w, gy = _inputs(cfg, seed)
    ws = ws or ConvWorkspace([cfg])
    xd, wd, gyd = (torch.from_numpy(a).to(dev) for a in (x, w, gy))
    got = [ws.forward(xd, wd), ws.grad_input(gyd, wd), ws.grad_weight(gyd, xd)]
    torch.cuda.synchronize()
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    ref = [oracle.forward_direct(x64, w64), oracle.grad_input_direct(gy64, w64), oracle.grad_weight_direct(gy64, x64)]
    for g, r, tol in zip(got, ref, (1e-4, 1e-4, 1e-3)):
        g = g.cpu().numpy()
        assert g.shape == r.shape
        assert oracle.rel_l2_error(g, r) <= 1e-4
        assert oracle.max_rel_error(g, r) <= tol


@pytest.mark.parametrize("cfg", [(11, 128, 3, 8, 2), (5, 100, 4, 6, 3), (3, 65, 2, 3, 2), (1, 128, 2, 2, 1),
                                 (128, 128, 2, 3, 2), (33, 96, 3, 5, 2)])
def test_ops_m128_vs_direct(dev, gemm_kind, cfg):
    _check_ops(LayerConfig(*cfg), 4000 + sum(cfg), dev)


def test_ops_m128_chunked_scratch(dev, monkeypatch):
    """1 MiB of scratch: every chunk is one operand row (several launches
    per transform); results must not change."""
    monkeypatch.setenv("FFTCONV_B200_LSCRATCH_MB", "1")
    _check_ops(LayerConfig(7, 128, 16, 8, 4), 4100, dev)


@pytest.mark.parametrize("cfg", [(11, 128, 3, 5, 7), (9, 120, 6, 4, 5)])
def test_ops_m128_narrow_kpad_chunked_rows(dev, monkeypatch, cfg):
    """A narrow kpad (f <= 8: 4 or 8) packs 16 / kpad operand rows into one
    K1b CTA; with 1 MiB of scratch the chunks hold a few rows each, so CTAs
    straddle chunk ends (rows past the chunk must be neither read nor
    written) and the batch is not a multiple of the rows per CTA."""
    monkeypatch.setenv("FFTCONV_B200_LSCRATCH_MB", "1")
    _check_ops(LayerConfig(*cfg), 4300 + sum(cfg), dev)


def test_ops_m128_reused_workspace_with_smaller_layers(dev):
    """One workspace serving m = 128 and m = 32 layers (conv_fft_test.cpp:191-209)."""
    big, small = LayerConfig(11, 128, 3, 8, 2), LayerConfig(5, 32, 4, 4, 2)
    ws = ConvWorkspace([big, small])
    _check_ops(small, 4200, dev, ws)
    _check_ops(big, 4201, dev, ws)
    _check_ops(small, 4202, dev, ws)


def test_m256_is_a_size_error(dev):
    import torch

    cfg = LayerConfig(3, 129, 1, 1, 1)
    ws = ConvWorkspace([cfg])
    x = torch.zeros((1, 1, 129, 129), device=dev)
    w = torch.zeros((1, 1, 3, 3), device=dev)
    with pytest.raises(SizeError):
        ws.forward(x, w)
