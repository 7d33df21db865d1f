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


@pytest.mark.parametrize("kind", ["tf32x3", "auto"])
def test_samples_of_very_different_magnitude(dev, kind):
    """Samples 1e-12 and 1e12 in one minibatch each keep their own relative
    accuracy under 3xTF32 and under auto (which falls back to 3xTF32 when
    rows span more than 2^18)."""
    from paper_1312_5851_b200 import _native

    cfg = LayerConfig(3, 8, 128, 128, 128)  # tensor-bound GEMM shape: auto launches the pair
    x, w, gy = _inputs(cfg, 93)
    for arr in (x, gy):
        arr[0] *= np.float32(1e12)
        arr[2] *= np.float32(1e-12)
    prev = _native.set_gemm_kind(kind)
    try:
        got = _run(cfg, x, w, gy, dev)
    finally:
        _native.set_gemm_kind(prev)
    ref = _ref(x, w, gy)
    for b in (0, 1, 2, 77):  # fprop / bprop outputs per sample
        for g, r in zip(got[:2], ref[:2]):
            assert oracle.rel_l2_error(g[b], r[b]) <= 1e-4
    assert oracle.rel_l2_error(got[2], ref[2]) <= 1e-4


def test_auto_route_selection(dev):
    """auto: 3xTF32 where the GEMM is byte-bound (P's shape); on a
    tensor-bound shape fp16x3 for well-scaled data and the 3xTF32 fallback
    when an operand's rows span more than 2^18."""
    import torch

    from paper_1312_5851_b200 import _native

    prev = _native.set_gemm_kind("auto")
    try:
        cfg = LayerConfig(3, 8, 128, 128, 128)  # MNK / (MK + NK + MN) = 42.7 > 42
        x, w, gy = _inputs(cfg, 94)
        ws = ConvWorkspace([cfg])
        xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
        y = ws.forward(xd, wd)
        assert ws.last_gemm_path() == "f16x3"
        assert oracle.rel_l2_error(y.cpu().numpy(), _ref(x, w, gy)[0]) <= 1e-4
        x2 = x.copy()
        x2[5] *= np.float32(2.0 ** -30)
        y2 = ws.forward(torch.from_numpy(x2).to(dev), wd)
        assert ws.last_gemm_path() == "tf32x3"
        r2 = _ref(x2, w, gy)[0]
        assert oracle.rel_l2_error(y2[5].cpu().numpy(), r2[5]) <= 1e-4
        p = LayerConfig(7, 32, 96, 96, 16)  # P-like shape (34.9): byte-bound
        xp, wp, _ = _inputs(p, 95)
        ConvWorkspace([p]).forward(torch.from_numpy(xp).to(dev), torch.from_numpy(wp).to(dev))
        wsp = ConvWorkspace([p])
        wsp.forward(torch.from_numpy(xp).to(dev), torch.from_numpy(wp).to(dev))
        assert wsp.last_gemm_path() == "tf32x3"
    finally:
        _native.set_gemm_kind(prev)
