"""Operator-level parity under both K3 precision schemes (fp16x3 default,
3xTF32 alternative; include/fftconv_b200.h fftconv_b200_set_gemm_kind):
full outputs vs the fp64 direct oracle at the reference's rel-L2 1e-4 bar,
including input magnitudes far outside fp16's range."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig

pytestmark = pytest.mark.gpu


def _run(cfg, x, w, gy, dev):
    import torch

    ws = ConvWorkspace([cfg])
    xd, wd, gyd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, w, gy))
    out = ws.forward(xd, wd), ws.grad_input(gyd, wd), ws.grad_weight(gyd, xd)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in out]


def _inputs(cfg, seed, sx=1.0, sw=1.0, sg=1.0):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT) * np.float32(sx)
    w = oracle.fill_uniform((fo, f, k, k), seed, oracle.ROLE_WEIGHTS) * np.float32(sw)
    gy = oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT) * np.float32(sg)
    return x, w, gy


def _ref(x, w, gy):
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    return (oracle.forward_direct(x64, w64), oracle.grad_input_direct(gy64, w64),
            oracle.grad_weight_direct(gy64, x64))


@pytest.mark.parametrize("cfg", [(5, 32, 16, 16, 8), (7, 32, 96, 96, 4), (3, 16, 40, 24, 130), (11, 64, 24, 20, 3),
                                 (3, 8, 5, 7, 3), (2, 4, 3, 2, 2), (2, 2, 3, 3, 2)])
def test_ops_vs_direct(dev, gemm_kind, cfg):
    cfg = LayerConfig(*cfg)
    x, w, gy = _inputs(cfg, 91)
    for g, r in zip(_run(cfg, x, w, gy, dev), _ref(x, w, gy)):
        assert oracle.rel_l2_error(g, r) <= 1e-4


@pytest.mark.parametrize("sx,sw,sg", [(1e-20, 1e10, 1e-15), (1e18, 1e-3, 1e12), (2.0 ** -100, 2.0 ** 60, 1.0)])
def test_ops_extreme_magnitudes(dev, gemm_kind, sx, sw, sg):
    cfg = LayerConfig(5, 16, 12, 10, 6)
    x, w, gy = _inputs(cfg, 92, sx, sw, sg)
    for g, r in zip(_run(cfg, x, w, gy, dev), _ref(x, w, gy)):
        assert np.isfinite(g).all()
        assert oracle.rel_l2_error(g, r) <= 1e-4


def test_kinds_agree_at_paper_point(dev):
    """fp16x3 and 3xTF32 agree to fp32 level at BASELINE configs[1]."""
    from paper_1312_5851_b200 import _native

    cfg = LayerConfig(7, 32, 96, 96, 128)
    x, w, gy = _inputs(cfg, 1234)
    lib = _native.lib()
    prev = lib.fftconv_b200_set_gemm_kind(0)
    try:
        a = _run(cfg, x, w, gy, dev)
        lib.fftconv_b200_set_gemm_kind(1)
        b = _run(cfg, x, w, gy, dev)
    finally:
        lib.fftconv_b200_set_gemm_kind(prev)
    for u, v in zip(a, b):
        assert oracle.rel_l2_error(u, v.astype(np.float64)) <= 1e-5
