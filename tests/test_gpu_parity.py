"""Operator-level parity of the B200 path against the CPU oracle.

Mirrors the reference's own hot-path tests (tests/conv_fft_test.cpp,
acceptance_test.cpp criteria 1/4/6) and adds the BASELINE.json shapes:
* small C config and random verify sweep: full outputs vs fp64 direct oracle;
* paper point P: full outputs vs the fp64 FFT oracle (== reference
  ConvWorkspace<double>, see test_oracle_golden.py);
* kernel/input sweep and the wide layer: sampled planes vs the fp64 direct
  oracle plus size-independent properties (adjoint triple, linearity, batch
  decomposability).
Bar (BASELINE.json north_star): max relative L2 error <= 1e-4 in fp32; the
reference's own f32 sup-norm tolerances 1e-4/1e-4/1e-3 (acceptance_test.cpp:47)
are checked too.
"""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import (CapacityError, ConfigError, ConvWorkspace, LayerConfig, ShapeError,
                                  SizeError, forward_fft, grad_input_fft, grad_weight_fft, workspace_for)

pytestmark = pytest.mark.gpu

L2_TOL = 1e-4


def _inputs(cfg, seed, dtype=np.float32):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT, dtype=dtype)
    w = oracle.fill_uniform((fo, f, k, k), seed, oracle.ROLE_WEIGHTS, dtype=dtype)
    gy = oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT, dtype=dtype)
    return x, w, gy


def _run_all(ws, x, w, gy, dev):
    import torch

    xd, wd, gyd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, w, gy))
    y = ws.forward(xd, wd)
    gx = ws.grad_input(gyd, wd)
    gw = ws.grad_weight(gyd, xd)
    torch.cuda.synchronize()
    return y.cpu().numpy(), gx.cpu().numpy(), gw.cpu().numpy()


def _direct64(x, w, gy):
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    return (oracle.forward_direct(x64, w64), oracle.grad_input_direct(gy64, w64),
            oracle.grad_weight_direct(gy64, x64))


def _assert_close(got, ref, sup_tols=(1e-4, 1e-4, 1e-3)):
    for g, r, tol in zip(got, ref, sup_tols):
        assert g.shape == r.shape
        assert oracle.rel_l2_error(g, r) <= L2_TOL
        assert oracle.max_rel_error(g, r) <= tol


# ------------------------------------------------- conv_fft_test.cpp:57-75
@pytest.mark.parametrize("cfg,seed", [((3, 16, 4, 6, 2), 21), ((5, 16, 4, 4, 2), 22), ((7, 32, 3, 5, 1), 23),
                                      ((1, 7, 2, 3, 2), 14), ((4, 9, 1, 1, 3), 15),
                                      ((3, 8, 2, 2, 2), 31), ((8, 8, 1, 2, 1), 32)])
def test_matches_direct_mixed_configs(dev, cfg, seed):
    cfg = LayerConfig(*cfg)
    x, w, gy = _inputs(cfg, seed)
    ws = ConvWorkspace([cfg])
    got = _run_all(ws, x, w, gy, dev)
    ref = _direct64(x, w, gy)
    # the reference's f32 bound is 1e-4 sup-norm for every op here (conv_fft_test.cpp:65-69)
    _assert_close(got, ref, (1e-4, 1e-4, 1e-4))


@pytest.mark.parametrize("cfg", [(3, 32, 24, 20, 3), (7, 30, 17, 33, 2), (8, 32, 5, 6, 4)])
def test_small_src_k1_at_m32_vs_direct(dev, monkeypatch, cfg):
    """The small-plane K1 (fft_small.cuh) at m = 32 (off by default, measured
    slower there; FFTCONV_B200_SMALLSRC32_MIN enables it), forced on for
    every small-plane operand here."""
    monkeypatch.setenv("FFTCONV_B200_SMALLSRC32_MIN", "1")
    cfg = LayerConfig(*cfg)
    x, w, gy = _inputs(cfg, 4400 + cfg.kernel)
    got = _run_all(ConvWorkspace([cfg]), x, w, gy, dev)
    _assert_close(got, _direct64(x, w, gy))


# ------------------------------------------------- BASELINE configs[0]
def test_small_cpu_config_vs_direct_oracle(dev):
    cfg = LayerConfig(kernel=5, image=32, in_maps=16, out_maps=16, batch=8)
    x, w, gy = _inputs(cfg, 1234)
    got = _run_all(ConvWorkspace([cfg]), x, w, gy, dev)
    _assert_close(got, _direct64(x, w, gy))


# ------------------------------------------------- reoriented GEMM (small batch)
@pytest.mark.parametrize("cfg", [(7, 32, 96, 96, 16), (5, 16, 40, 24, 3), (11, 64, 64, 48, 8),
                                 (3, 12, 33, 20, 5)])
def test_small_batch_swapped_gemm_vs_direct(dev, cfg):
    """Batches smaller than the maps run the per-bin GEMM transposed (maps on
    the 128-row tile, conjugated epilogue, K4 reading the transposed product);
    the results must not change (fprop / bprop; accGrad is unaffected)."""
    cfg = LayerConfig(*cfg)
    x, w, gy = _inputs(cfg, 77)
    got = _run_all(ConvWorkspace([cfg]), x, w, gy, dev)
    _assert_close(got, _direct64(x, w, gy))


# ------------------------------------------------- known answers
def test_unit_kernel_is_identity(dev):
    """conv_fft_test.cpp:77-85"""
    import torch

    x = oracle.fill_uniform((2, 2, 6, 6), 41, oracle.ROLE_INPUT)
    w = np.zeros((2, 2, 1, 1), dtype=np.float32)
    w[0, 0, 0, 0] = 1
    w[1, 1, 0, 0] = 1
    ws = ConvWorkspace([(1, 6, 2, 2, 2)])
    y = ws.forward(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)).cpu().numpy()
    assert oracle.max_rel_error(y, x) < 1e-6


def test_zero_kernel_gives_zero(dev):
    """conv_fft_test.cpp:87-93"""
    import torch

    x = oracle.fill_uniform((1, 2, 5, 5), 42, oracle.ROLE_INPUT)
    w = np.zeros((3, 2, 2, 2), dtype=np.float32)
    ws = ConvWorkspace([(2, 5, 2, 3, 1)])
    y = ws.forward(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)).cpu().numpy()
    assert np.abs(y).max() < 1e-7


@pytest.mark.parametrize("n,k,u0,v0", [(8, 3, 1, 2), (32, 7, 6, 0), (32, 7, 0, 6), (64, 11, 3, 9), (13, 4, 2, 3)])
def test_corner_impulse_selects_shifted_window(dev, n, k, u0, v0):
    """conv_fft_test.cpp:95-107: catches conj / transpose / mirror mistakes."""
    import torch

    x = oracle.fill_uniform((1, 1, n, n), 43, oracle.ROLE_INPUT)
    w = np.zeros((1, 1, k, k), dtype=np.float32)
    w[0, 0, u0, v0] = 1
    ws = ConvWorkspace([(k, n, 1, 1, 1)])
    y = ws.forward(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)).cpu().numpy()
    no = n - k + 1
    assert np.abs(y[0, 0] - x[0, 0, u0:u0 + no, v0:v0 + no]).max() < 1e-5


@pytest.mark.parametrize("n,no,i0,j0", [(6, 2, 1, 1), (32, 26, 3, 20), (16, 4, 0, 3)])
def test_grad_weight_impulse_extracts_input_window(dev, n, no, i0, j0):
    """conv_fft_test.cpp:109-119"""
    import torch

    x = oracle.fill_uniform((1, 1, n, n), 44, oracle.ROLE_INPUT)
    gy = np.zeros((1, 1, no, no), dtype=np.float32)
    gy[0, 0, i0, j0] = 1
    k = n - no + 1
    ws = ConvWorkspace([(k, n, 1, 1, 1)])
    gw = ws.grad_weight(torch.from_numpy(gy).to(dev), torch.from_numpy(x).to(dev)).cpu().numpy()
    assert gw.shape == (1, 1, k, k)
    assert np.abs(gw[0, 0] - x[0, 0, i0:i0 + k, j0:j0 + k]).max() < 1e-5


def test_grad_input_delta_reproduces_kernel(dev):
    """SPEC conv-direct example: gy = [1] (1x1) -> gx == w."""
    import torch

    w = np.array([[[[1, 2], [3, 4]]]], dtype=np.float32)
    gy = np.ones((1, 1, 1, 1), dtype=np.float32)
    ws = ConvWorkspace([(2, 2, 1, 1, 1)])
    gx = ws.grad_input(torch.from_numpy(gy).to(dev), torch.from_numpy(w).to(dev)).cpu().numpy()
    assert np.abs(gx - w).max() < 1e-6


def test_box_kernel_hand_example(dev):
    """conv_direct_test.cpp:31-44: [[1,2,3],[4,5,6],[7,8,9]] * ones(2x2) = [[12,16],[24,28]]."""
    import torch

    x = np.arange(1, 10, dtype=np.float32).reshape(1, 1, 3, 3)
    w = np.ones((1, 1, 2, 2), dtype=np.float32)
    ws = ConvWorkspace([(2, 3, 1, 1, 1)])
    y = ws.forward(torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)).cpu().numpy()
    assert np.abs(y[0, 0] - np.array([[12, 16], [24, 28]])).max() < 1e-5


# ------------------------------------------------- properties
def test_adjoint_triple(dev):
    """conv_fft_test.cpp:121-140 (fp32 here: 1e-5 instead of the f64 1e-8)."""
    ws = ConvWorkspace([(4, 12, 4, 4, 3)])
    for s in range(8):
        S, f, fp = 1 + s % 3, 1 + s % 4, 1 + (s + 2) % 4
        n, k = 5 + s % 8, 1 + s % 4
        cfg = LayerConfig(k, n, f, fp, S)
        x, w, gy = _inputs(cfg, s)
        y, gx, gw = _run_all(ws, x, w, gy, dev)
        a = float(np.dot(y.ravel().astype(np.float64), gy.ravel()))
        b = float(np.dot(x.ravel().astype(np.float64), gx.ravel()))
        c = float(np.dot(w.ravel().astype(np.float64), gw.ravel()))
        scale = max(abs(a), abs(b), abs(c), 1e-30)
        assert abs(a - b) / scale < 1e-5
        assert abs(a - c) / scale < 1e-5


def test_counters_match_plan_and_are_kernel_invariant(dev):
    """conv_fft_test.cpp:211-253 / acceptance criterion 6."""
    n, S, f, fp = 16, 2, 3, 4
    bins = 16 * 9
    seen = None
    for k in (3, 5, 7, 11):
        cfg = LayerConfig(k, n, f, fp, S)
        ws = ConvWorkspace([cfg])
        x, w, gy = _inputs(cfg, 70)
        import torch

        xd, wd, gyd = (torch.from_numpy(a).to(dev) for a in (x, w, gy))
        ws.forward(xd, wd)
        fwd = ws.counters()
        assert fwd == (S * f + fp * f, S * fp, bins * fp * f * S)
        ws.reset_counters()
        ws.grad_input(gyd, wd)
        gin = ws.counters()
        assert gin == (S * fp + fp * f, S * f, bins * fp * f * S)
        ws.reset_counters()
        ws.grad_weight(gyd, xd)
        gwc = ws.counters()
        assert gwc == (S * f + S * fp, fp * f, bins * fp * f * S)
        if seen is not None:
            assert (fwd, gin, gwc) == seen
        seen = (fwd, gin, gwc)


def test_reuse_across_layers_is_bit_stable(dev):
    """conv_fft_test.cpp:191-209"""
    import torch

    a = LayerConfig(3, 6, 2, 3, 2)
    b = LayerConfig(5, 12, 3, 2, 1)
    ws = ConvWorkspace([a, b])
    xa, wa, _ = _inputs(a, 60)
    xb, wb, _ = _inputs(b, 62)
    t = lambda v: torch.from_numpy(v).to(dev)  # noqa: E731
    first = ws.forward(t(xa), t(wa)).cpu().numpy()
    ws.forward(t(xb), t(wb))
    again = ws.forward(t(xa), t(wa)).cpu().numpy()
    assert np.array_equal(first, again)


def test_thread_count_does_not_change_bits(dev):
    """conv_fft_test.cpp:255-277: `threads` is accepted and results are bit-identical."""
    cfg = LayerConfig(3, 10, 3, 4, 2)
    x, w, gy = _inputs(cfg, 80)
    base = ConvWorkspace([cfg])
    r1 = (base.forward(x, w, 1), base.grad_input(gy, w, 1), base.grad_weight(gy, x, 1))
    for threads in (2, 3, 7):
        ws = ConvWorkspace([cfg])
        r2 = (ws.forward(x, w, threads), ws.grad_input(gy, w, threads), ws.grad_weight(gy, x, threads))
        for p, q in zip(r1, r2):
            assert np.array_equal(p, q)


def test_free_function_wrappers_host_path(dev):
    """conv_fft_test.cpp:279-294, through the host-pointer (drop-in) entry points."""
    cfg = LayerConfig(2, 5, 1, 2, 1)
    ws = workspace_for([cfg])
    x, w, gy = _inputs(cfg, 90)
    got = (forward_fft(ws, x, w), grad_input_fft(ws, gy, w), grad_weight_fft(ws, gy, x))
    _assert_close(got, _direct64(x, w, gy), (1e-5, 1e-5, 1e-5))


# ------------------------------------------------- error contract
def test_workspace_capacities(dev):
    """conv_fft_test.cpp:142-161"""
    cfg = LayerConfig(3, 8, 2, 5, 1)
    ws = ConvWorkspace([cfg])
    assert ws.max_fft_size() == 8
    assert (ws.capacity_x(), ws.capacity_w(), ws.capacity_y()) == (40 * 1 * 2, 40 * 5 * 2, 40 * 1 * 5)
    assert ws.frequency_bytes() == (80 + 400 + 200) * 8
    ws2 = ConvWorkspace([LayerConfig(3, 8, 2, 5, 1), LayerConfig(3, 8, 4, 1, 3)])
    assert (ws2.capacity_x(), ws2.capacity_w(), ws2.capacity_y()) == (40 * 3 * 4, 40 * 5 * 2, 40 * 1 * 5)


def test_error_contract(dev):
    """conv_fft_test.cpp:163-189, on both device and host entry points."""
    import torch

    with pytest.raises(ConfigError):
        ConvWorkspace([])
    ws = ConvWorkspace([(3, 8, 2, 2, 1)])
    w = oracle.fill_uniform((2, 2, 3, 3), 50, 2)
    for to in (lambda a: a, lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)):
        with pytest.raises(CapacityError):
            ws.forward(to(oracle.fill_uniform((2, 2, 8, 8), 51, 1)), to(w))
        with pytest.raises(CapacityError):
            ws.forward(to(oracle.fill_uniform((1, 2, 9, 9), 52, 1)), to(w))
        x = to(oracle.fill_uniform((1, 2, 8, 8), 53, 1))
        with pytest.raises(ShapeError):
            ws.forward(x, to(np.zeros((2, 3, 3, 3), np.float32)))
        with pytest.raises(SizeError):
            ws.forward(x, to(np.zeros((2, 2, 9, 9), np.float32)))
        with pytest.raises(SizeError):
            ws.forward(to(np.zeros((1, 2, 8, 6), np.float32)), to(np.zeros((2, 2, 3, 3), np.float32)))
        gy = to(oracle.fill_uniform((1, 2, 6, 6), 54, 3))
        with pytest.raises(ShapeError):
            ws.grad_input(gy, to(np.zeros((3, 2, 3, 3), np.float32)))
        with pytest.raises(ShapeError):
            ws.grad_weight(to(np.zeros((2, 2, 6, 6), np.float32)), x)
        with pytest.raises(SizeError):
            ws.grad_weight(to(np.zeros((1, 2, 9, 9), np.float32)), x)


# ------------------------------------------------- acceptance criterion 1
def test_random_verify_sweep_100_configs(dev):
    """acceptance_test.cpp:42-55: 100 random configs (seed 2024), one reused
    workspace, f32 tolerances 1e-4 / 1e-4 / 1e-3 vs the direct oracle."""
    cfgs = [LayerConfig(*c) for c in oracle.random_verify_configs(100, 2024)]
    ws = ConvWorkspace(cfgs)
    worst = [0.0, 0.0, 0.0]
    for cfg in cfgs:
        x, w, gy = _inputs(cfg, 2024)
        got = _run_all(ws, x, w, gy, dev)
        ref = _direct64(x, w, gy)
        for i in range(3):
            worst[i] = max(worst[i], oracle.max_rel_error(got[i], ref[i]))
            assert oracle.rel_l2_error(got[i], ref[i]) <= L2_TOL
    assert worst[0] <= 1e-4 and worst[1] <= 1e-4 and worst[2] <= 1e-3, worst


# ------------------------------------------------- BASELINE configs[1]
def test_paper_point_full_vs_fft_oracle(dev):
    """S=128, f=f'=96, n=32, k=7: every output vs the fp64 FFT oracle."""
    cfg = LayerConfig(7, 32, 96, 96, 128)
    x, w, gy = _inputs(cfg, 1234)
    got = _run_all(ConvWorkspace([cfg]), x, w, gy, dev)
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    ref = (oracle.forward_fft(x64, w64), oracle.grad_input_fft(gy64, w64), oracle.grad_weight_fft(gy64, x64))
    _assert_close(got, ref)


def _assert_adjoint(x, w, gy, y, gx, gw, tol):
    """<y,gy> = <x,gx> = <w,gw>, gaps relative to the Cauchy-Schwarz bound
    (the dot products themselves cancel heavily at these sizes)."""
    d = lambda a, b: float(np.dot(a.ravel().astype(np.float64), b.ravel().astype(np.float64)))  # noqa: E731
    nrm = lambda a: float(np.linalg.norm(a.ravel().astype(np.float64)))  # noqa: E731
    a, b, c = d(y, gy), d(x, gx), d(w, gw)
    scale = max(nrm(y) * nrm(gy), nrm(x) * nrm(gx), nrm(w) * nrm(gw))
    assert abs(a - b) / scale < tol and abs(a - c) / scale < tol, (a, b, c, scale)


def _sampled_planes_check(dev, cfg, seed, nplanes=6):
    import torch

    x, w, gy = _inputs(cfg, seed)
    ws = ConvWorkspace([cfg])
    y, gx, gw = _run_all(ws, x, w, gy, dev)
    rng = np.random.default_rng(seed)
    S, f, fo = cfg.batch, cfg.in_maps, cfg.out_maps
    ids_y = rng.choice(S * fo, nplanes, replace=False)
    ids_gx = rng.choice(S * f, nplanes, replace=False)
    ids_gw = rng.choice(fo * f, nplanes, replace=False)
    x64, w64, gy64 = (a.astype(np.float64) for a in (x, w, gy))
    ry = oracle.forward_direct_planes(x64, w64, ids_y)
    rgx = oracle.grad_input_direct_planes(gy64, w64, ids_gx)
    rgw = oracle.grad_weight_direct_planes(gy64, x64, ids_gw)
    gy_ = y.reshape(S * fo, *y.shape[2:])[ids_y]
    ggx = gx.reshape(S * f, *gx.shape[2:])[ids_gx]
    ggw = gw.reshape(fo * f, *gw.shape[2:])[ids_gw]
    for got, ref in ((gy_, ry), (ggx, rgx), (ggw, rgw)):
        assert oracle.rel_l2_error(got, ref) <= L2_TOL
    # adjoint triple over the full tensors (size-independent property)
    _assert_adjoint(x, w, gy, y, gx, gw, 1e-6)
    del torch


@pytest.mark.parametrize("n", [16, 32, 64])
@pytest.mark.parametrize("k", [3, 5, 7, 9, 11, 13])
def test_kernel_input_sweep_sampled(dev, n, k):
    """BASELINE configs[2]: S=128, f=f'=96, n in {16,32,64}, k in {3..13}."""
    _sampled_planes_check(dev, LayerConfig(k, n, 96, 96, 128), 1234 + n + k)


def test_wide_layer_sampled(dev):
    """BASELINE configs[3] at one GPU: S=128, f=f'=256, n=64, k=11."""
    _sampled_planes_check(dev, LayerConfig(11, 64, 256, 256, 128), 1234, nplanes=4)


def test_batch_decomposability(dev):
    """conv_direct_test.cpp:186-212: y/gx concatenate over the batch, gw sums --
    the property S-sharding relies on."""
    cfg = LayerConfig(5, 16, 6, 7, 8)
    x, w, gy = _inputs(cfg, 5)
    ws = ConvWorkspace([cfg])
    y, gx, gw = _run_all(ws, x, w, gy, dev)
    parts = [_run_all(ws, x[i:i + 2], w, gy[i:i + 2], dev) for i in range(0, 8, 2)]
    assert oracle.max_rel_error(np.concatenate([p[0] for p in parts]), y) < 1e-6
    assert oracle.max_rel_error(np.concatenate([p[1] for p in parts]), gx) < 1e-6
    assert oracle.max_rel_error(sum(p[2] for p in parts), gw) < 1e-5
