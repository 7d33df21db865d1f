"""Workspace reuse across layers, streams and GEMM kinds (round-1 advisor
findings): a layer with more operand rows than any registered config, a
device-path call followed by a host-path call on the same workspace, and the
per-workspace GEMM precision override.  Reference contract: one workspace
serves every registered layer in any order (conv_fft.hpp:43-72, :211-222)."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig

pytestmark = pytest.mark.gpu


def _inputs(cfg, seed):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT)
    w = oracle.fill_uniform((fo, f, k, k), seed, oracle.ROLE_WEIGHTS)
    gy = oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT)
    return x, w, gy


def _fft64(x, w, gy):
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    return oracle.forward_fft(x64, w64), oracle.grad_input_fft(gy64, w64), oracle.grad_weight_fft(gy64, x64)


@pytest.mark.parametrize("kind", ["f16x3", "auto", "tf32x3"])
def test_more_operand_rows_than_registered(dev, kind):
    """Registered: n=64, f=f'=32, S=16 (32 operand rows).  Called: n=16,
    S=150, f=f'=40 -- inside every capacity, but 150 rows of K1 per-row
    maxima: the words grow instead of overrunning."""
    import torch

    ws = ConvWorkspace([LayerConfig(5, 64, 32, 32, 16)])
    ws.set_gemm_kind(kind)
    cfg = LayerConfig(5, 16, 40, 40, 150)
    x, w, gy = _inputs(cfg, 41)
    x[7] *= 1e3  # one sample far larger than the rest: row maxima matter
    xd, wd, gyd = (torch.from_numpy(a).to(dev) for a in (x, w, gy))
    got = (ws.forward(xd, wd), ws.grad_input(gyd, wd), ws.grad_weight(gyd, xd))
    torch.cuda.synchronize()
    for g, r in zip(got, _fft64(x, w, gy)):
        assert oracle.rel_l2_error(g.cpu().numpy(), r) <= 1e-4


def test_device_then_host_call_ordered(dev):
    """A device-path operator on a side stream followed at once by a host-path
    operator on the same workspace (shared spectra buffers; ADVICE r1,
    medium): both results must be right."""
    import torch

    cfg = LayerConfig(7, 32, 96, 96, 128)
    ws = ConvWorkspace([cfg])
    x, w, gy = _inputs(cfg, 42)
    ref = _fft64(x, w, gy)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    side = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(side):
            torch.cuda._sleep(2_000_000)  # keep the side stream busy: the race window
            y_dev = ws.forward(xd, wd)
        gx_host = ws.grad_input(gy, w)  # numpy: the host entry point, its own stream
        torch.cuda.synchronize()
        assert oracle.rel_l2_error(y_dev.cpu().numpy(), ref[0]) <= 1e-4
        assert oracle.rel_l2_error(gx_host, ref[1]) <= 1e-4


def test_per_workspace_gemm_kind(dev):
    """Two workspaces in one process with different K3 schemes."""
    import torch

    cfg = LayerConfig(3, 16, 64, 64, 128)
    a, b = ConvWorkspace([cfg]), ConvWorkspace([cfg])
    assert a.set_gemm_kind("f16x3") is None
    assert b.set_gemm_kind("tf32x3") is None
    x, w, gy = _inputs(cfg, 43)
    xd, wd = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
    ya = a.forward(xd, wd)
    assert a.last_gemm_path() == "f16x3"
    yb = b.forward(xd, wd)
    assert b.last_gemm_path() == "tf32x3"
    ref = _fft64(x, w, gy)[0]
    for y in (ya, yb):
        assert oracle.rel_l2_error(y.cpu().numpy(), ref) <= 1e-4
    assert a.set_gemm_kind(None) == "f16x3"


def test_live_spans_cover_each_kernel(dev):
    """fftconv_b200_set_span_timing: every operator's K1 / K3 / K4 span is
    recorded, positive, and together no longer than the operator's event
    time (the spans exclude the launch hand-offs)."""
    import torch

    cfg = LayerConfig(7, 32, 48, 40, 32)
    ws = ConvWorkspace([cfg])
    x, w, gy = _inputs(cfg, 44)
    xd, wd, gyd = (torch.from_numpy(a).to(dev) for a in (x, w, gy))
    ws.forward(xd, wd)
    ws.set_span_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ws.forward(xd, wd)
    ws.grad_input(gyd, wd)
    ws.grad_weight(gyd, xd)
    b.record()
    spans = ws.span_ms()
    ws.set_span_timing(False)
    assert len(spans) == 3
    for sp in spans:
        assert all(v is not None and v > 0 for v in sp), spans
    assert sum(sum(sp) for sp in spans) <= a.elapsed_time(b) * 1.05
