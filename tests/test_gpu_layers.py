"""Layer-stack stages and one full training iteration on the GPU against the
reference (layers.hpp): relu / max-pool / fit_to kernels vs numpy
restatements of layers.hpp:34-109 and :393-407, and run_iteration on the
reference-net-small preset vs the reference's own run_iteration (FFT engine)
on identical parameters and batch."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import layers

pytestmark = pytest.mark.gpu


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def test_relu(dev):
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 5, 7, 9)).astype(np.float32)   # 945 elements: vector body + tail
    gy = rng.standard_normal(x.shape).astype(np.float32)
    xd = _t(x, dev)
    assert np.array_equal(layers.relu_forward(xd).cpu().numpy(), np.where(x > 0, x, 0))
    assert np.array_equal(layers.relu_backward(_t(gy, dev), xd).cpu().numpy(), np.where(x > 0, gy, 0))


@pytest.mark.parametrize("S,f,fo,n,k", [
    (4, 3, 8, 16, 5),     # m = 16
    (4, 6, 10, 30, 3),    # m = 32
    (3, 5, 7, 16, 13),    # small output crop (direct-DFT K4 path)
    (2, 4, 6, 60, 5),     # m = 64
    (2, 3, 4, 118, 11),   # m = 128 (two-pass K4)
    (2, 2, 3, 2, 1),      # m = 2 plane kernels
])
def test_forward_relu_fused_equals_relu_of_forward(dev, S, f, fo, n, k):
    """fftconv_b200_forward_relu: the stack's relu fused into K4's stores
    is bit-identical to forward followed by the relu kernel."""
    from paper_1312_5851_b200 import ConvWorkspace, LayerConfig

    rng = np.random.default_rng(S * 1000 + n)
    x = _t(rng.standard_normal((S, f, n, n)).astype(np.float32), dev)
    w = _t(rng.standard_normal((fo, f, k, k)).astype(np.float32), dev)
    ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
    y = ws.forward(x, w)
    yr = ws.forward(x, w, relu=True)
    assert (y > 0).any() and (y < 0).any()
    assert np.array_equal(yr.cpu().numpy(), layers.relu_forward(y).cpu().numpy())


@pytest.mark.parametrize("S,f,fo,pre,n,k", [
    (4, 5, 6, 13, 16, 3),     # m = 16
    (4, 6, 8, 30, 32, 3),     # m = 32 (AlexNet conv3-5)
    (2, 4, 6, 59, 64, 5),     # m = 64 (AlexNet conv2)
    (2, 3, 4, 100, 128, 11),  # m = 128
])
def test_fit_folded_operators_equal_fit_to_then_operator(dev, S, f, fo, pre, n, k):
    """forward_fit / grad_weight_fit on the pre x pre planes with the layer
    image n == the operators on fit_to(x, n); grad_input_fit(size=pre) ==
    fit_to(grad_input, pre)."""
    import torch

    from paper_1312_5851_b200 import ConvWorkspace, LayerConfig

    rng = np.random.default_rng(pre * 7 + n)
    x = _t(rng.standard_normal((S, f, pre, pre)).astype(np.float32), dev)
    w = _t(rng.standard_normal((fo, f, k, k)).astype(np.float32), dev)
    no = n - k + 1
    gy = _t(rng.standard_normal((S, fo, no, no)).astype(np.float32), dev)
    ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
    xp = layers.fit_to(x, n)
    pairs = [
        (ws.forward(x, w, image=n), ws.forward(xp, w)),
        (ws.forward(x, w, image=n, relu=True), layers.relu_forward(ws.forward(xp, w))),
        (ws.grad_input(gy, w, size=pre), layers.fit_to(ws.grad_input(gy, w), pre)),
        (ws.grad_weight(gy, x, image=n), ws.grad_weight(gy, xp)),
    ]
    torch.cuda.synchronize()
    for got, want in pairs:
        g, r = got.cpu().numpy(), want.cpu().numpy()
        assert g.shape == r.shape
        assert oracle.rel_l2_error(g, r) <= 1e-6


def test_maxpool_relu_backward_fused_equals_two_kernels(dev):
    """fftconv_b200_maxpool_relu_backward == relu_backward(maxpool_backward(g), x)
    for a pool fed by relu(x): windows of all zeros (relu'd negatives) and
    ties included."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3, 4, 10, 12)).astype(np.float32)
    x[0, 0, :4, :4] = -1.0        # an all-negative region: pooled value 0
    x[1, 1, 2:4, 2:4] = 0.5       # a tie
    xd = _t(x, dev)
    r = layers.relu_forward(xd)
    rec = layers.maxpool_forward(r)
    g = _t(rng.standard_normal(tuple(rec[0].shape)).astype(np.float32), dev)
    two = layers.relu_backward(layers.maxpool_backward(g, rec), xd).cpu().numpy()
    one = layers.maxpool_relu_backward(g, rec).cpu().numpy()
    assert np.array_equal(one, two)


def _pool_ref(x):
    S, M, R, Cc = x.shape
    y = np.zeros((S, M, R // 2, Cc // 2), np.float32)
    arg = np.zeros(y.shape, np.int64)
    for b in range(S):
        for m in range(M):
            for i in range(R // 2):
                for j in range(Cc // 2):
                    best = 2 * i * Cc + 2 * j
                    bv = x[b, m].reshape(-1)[best]
                    for di in range(2):
                        for dj in range(2):
                            p = (2 * i + di) * Cc + 2 * j + dj
                            if x[b, m].reshape(-1)[p] > bv:
                                bv, best = x[b, m].reshape(-1)[p], p
                    y[b, m, i, j], arg[b, m, i, j] = bv, best
    return y, arg


def test_maxpool(dev):
    rng = np.random.default_rng(2)
    x = rng.integers(-3, 3, (2, 3, 6, 8)).astype(np.float32)  # many ties: earliest element wins
    y_ref, arg_ref = _pool_ref(x)
    y, arg, shape = layers.maxpool_forward(_t(x, dev))
    assert np.array_equal(y.cpu().numpy(), y_ref)
    assert np.array_equal(arg.cpu().numpy(), arg_ref)
    gy = rng.standard_normal(y_ref.shape).astype(np.float32)
    gx = layers.maxpool_backward(_t(gy, dev), (y, arg, shape)).cpu().numpy()
    gx_ref = np.zeros_like(x)
    for b in range(2):
        for m in range(3):
            flat = gx_ref[b, m].reshape(-1)
            for i in range(3):
                for j in range(4):
                    flat[arg_ref[b, m, i, j]] += gy[b, m, i, j]
    assert np.array_equal(gx, gx_ref)


@pytest.mark.parametrize("size", [5, 8, 11])
def test_fit_to(dev, size):
    x = np.arange(2 * 3 * 8 * 8, dtype=np.float32).reshape(2, 3, 8, 8)
    got = layers.fit_to(_t(x, dev), size).cpu().numpy()
    ref = np.zeros((2, 3, size, size), np.float32)
    r = min(size, 8)
    ref[:, :, :r, :r] = x[:, :, :r, :r]
    assert np.array_equal(got, ref)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_run_iteration_matches_reference(dev):
    spec = layers.preset_network("reference-net-small")
    seed, S = 1234, spec.default_batch
    params = layers.init_params(spec, seed)
    batch = layers.make_batch(spec, S, seed)
    res = layers.run_iteration(spec, params, batch)
    ref_flat, ref = oracle.ref_run_iteration(spec.records(), S, seed, engine=1)
    assert res.grad_input_calls == int(ref["grad_input_calls"]) == 4
    # 5 fprop + 5 accGrad + 4 bprop operator calls (>= 3 launches each) + the layer stages
    assert res.gpu_launches >= 3 * (5 + 5 + 4)
    assert abs(res.loss - ref["loss"]) <= 1e-5 * abs(ref["loss"])
    off = 0
    for g in res.conv_weight_grads:
        n = g.numel()
        assert _rel(g.cpu().numpy().reshape(-1), ref_flat[off:off + n]) <= 1e-4
        off += n
    n = res.fc_weight_grad.numel()
    assert _rel(res.fc_weight_grad.cpu().numpy().reshape(-1), ref_flat[off:off + n]) <= 1e-5
    off += n
    assert _rel(res.fc_bias_grad.cpu().numpy(), ref_flat[off:]) <= 1e-6
    assert abs(res.grad_checksum - ref["grad_checksum"]) <= 1e-4 * abs(ref["grad_checksum"])
    assert res.times.total_ms() > 0


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
def test_alexnet128_iteration_matches_reference(dev):
    """BASELINE configs[4]'s stack (first layer n = 128: FFT size 128) at a
    small batch.  Five conv layers of fp32 backprop drift: the reference's
    own run_iteration<float> is 1.7e-3 from run_iteration<double> at layer 1
    (measured), so the bar is "no further from the fp64 reference than the
    reference's fp32 path", per layer."""
    spec = layers.preset_network("alexnet-128")
    seed, S = 77, 1
    params = layers.init_params(spec, seed)
    batch = layers.make_batch(spec, S, seed)
    res = layers.run_iteration(spec, params, batch)
    g32, r32 = oracle.ref_run_iteration(spec.records(), S, seed, engine=1)
    g64, r64 = oracle.ref_run_iteration(spec.records(), S, seed, engine=1, dtype=np.float64)
    assert res.grad_input_calls == int(r64["grad_input_calls"]) == 4
    assert abs(res.loss - r64["loss"]) <= 1e-4 * abs(r64["loss"])
    off = 0
    for g in res.conv_weight_grads:
        n = g.numel()
        ours = _rel(g.cpu().numpy().reshape(-1), g64[off:off + n])
        ref = _rel(g32[off:off + n], g64[off:off + n])
        assert ours <= max(ref, 1e-4), (ours, ref)
        off += n
