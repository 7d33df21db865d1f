"""Full-size parity at every BASELINE configuration the bench times: every
output element of the three operators, not sampled planes.

Golden: the reference's own ConvWorkspace<double> (oracle/_ref, built from
/root/reference by oracle/Makefile and shipped prebuilt), run on all host
threads; where that library is absent, the fp64 C restatement of the same
FFT path (oracle.forward_fft & co.; both are pinned to each other in
tests/test_oracle_golden.py).  Bar (BASELINE.json): relative L2 error <= 1e-4
over each whole tensor, plus the reference's f32 sup-norm tolerances
1e-4 / 1e-4 / 1e-3 (acceptance_test.cpp:42-55).

* BASELINE configs[3] (wide layer, S=128 f=f'=256 n=64 k=11) under each GEMM
  precision scheme -- 3xTF32 (the north star's), fp16x3 and auto;
* BASELINE configs[2], all 18 points (S=128 f=f'=96, n in {16,32,64},
  k in {3..13});
* the benched layer stacks (reference-net and alexnet-128 = configs[4]) at
  S=128 against the reference's run_iteration<double>.
"""
import functools

import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig, layers

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

L2_TOL = 1e-4
SUP_TOLS = (1e-4, 1e-4, 1e-3)


def _inputs(cfg, seed):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT)
    w = oracle.fill_uniform((fo, f, k, k), seed, oracle.ROLE_WEIGHTS)
    gy = oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT)
    return x, w, gy


@functools.lru_cache(maxsize=2)
def _golden(key, seed):
    """fp64 y, gx, gw of layer `key` = (k, n, f, f', S) on the generator's inputs."""
    cfg = LayerConfig(*key)
    x, w, gy = (a.astype(np.float64) for a in _inputs(cfg, seed))
    if oracle.ref_available():
        ws = oracle.RefWorkspace([key], dtype=np.float64)
        th = int(oracle.ref_lib().ref_resolve_threads(0))
        return ws.forward(x, w, th), ws.grad_input(gy, w, th), ws.grad_weight(gy, x, th)
    return oracle.forward_fft(x, w), oracle.grad_input_fft(gy, w), oracle.grad_weight_fft(gy, x)


def _run(ws, cfg, seed, dev):
    import torch

    x, w, gy = (torch.from_numpy(a).to(dev) for a in _inputs(cfg, seed))
    out = (ws.forward(x, w), ws.grad_input(gy, w), ws.grad_weight(gy, x))
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in out]


def _check(got, ref):
    errs = []
    for name, g, r, sup in zip(("y", "gx", "gw"), got, ref, SUP_TOLS):
        assert g.shape == r.shape, name
        assert np.isfinite(g).all(), name
        l2, mx = oracle.rel_l2_error(g, r), oracle.max_rel_error(g, r)
        errs.append((name, l2, mx))
        assert l2 <= L2_TOL, (name, l2)
        assert mx <= sup, (name, mx)
    return errs


@pytest.mark.parametrize("kind", ["tf32x3", "f16x3", "auto"])
def test_wide_layer_full(dev, kind):
    """BASELINE configs[3] on one GPU, every element, each GEMM scheme."""
    key = (11, 64, 256, 256, 128)
    ws = ConvWorkspace([LayerConfig(*key)])
    ws.set_gemm_kind(kind)
    got = _run(ws, LayerConfig(*key), 1234, dev)
    if kind != "auto":
        assert ws.last_gemm_path() == kind
    _check(got, _golden(key, 1234))


@pytest.mark.parametrize("n", [16, 32, 64])
@pytest.mark.parametrize("k", [3, 5, 7, 9, 11, 13])
def test_kernel_input_sweep_full(dev, n, k):
    """BASELINE configs[2]: S=128, f=f'=96, every element of every point."""
    key = (k, n, 96, 96, 128)
    got = _run(ConvWorkspace([LayerConfig(*key)]), LayerConfig(*key), 1234 + n + k, dev)
    _check(got, _golden(key, 1234 + n + k))


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("preset", ["reference-net", "alexnet-128"])
def test_stack_iteration_full_batch(dev, preset):
    """The benched stacks at their benched batch (S = 128) vs the
    reference's run_iteration<double>: loss, every conv weight gradient, fc
    gradients.  fp32 backprop through several conv layers drifts (the first
    layer's weight gradient is a 128-sample sum with heavy cancellation: the
    reference's own run_iteration<float> is ~1e-3 from fp64 there), and the
    drift is dominated by relu / max-pool decisions that any fp32 rounding
    flips (re-blocking one m = 64 kernel, with per-operator errors unchanged
    to three digits, moved alexnet-128's layer-2 ratio 1.85 -> 2.04), so the
    bar per tensor is "the same order as the reference's own fp32 path":
    within 3x of its distance from fp64, floored at the north star's 1e-4.
    Per-operator parity (the north star's bar) is checked element by element
    above."""
    spec = layers.preset_network(preset)
    seed, S = 1234, spec.default_batch
    assert S == 128
    params = layers.init_params(spec, seed)
    batch = layers.make_batch(spec, S, seed)
    res = layers.run_iteration(spec, params, batch)
    g32, r32 = oracle.ref_run_iteration(spec.records(), S, seed, engine=1)
    g64, r64 = oracle.ref_run_iteration(spec.records(), S, seed, engine=1, dtype=np.float64)
    assert res.grad_input_calls == int(r64["grad_input_calls"])
    assert abs(res.loss - r64["loss"]) <= max(3 * abs(r32["loss"] - r64["loss"]), 1e-5 * abs(r64["loss"]))
    off = 0
    tensors = [g.cpu().numpy().reshape(-1) for g in res.conv_weight_grads]
    tensors += [res.fc_weight_grad.cpu().numpy().reshape(-1), res.fc_bias_grad.cpu().numpy().reshape(-1)]
    rows = []
    for i, g in enumerate(tensors):
        n = g.size
        rows.append((i, _rel(g, g64[off:off + n]), _rel(g32[off:off + n], g64[off:off + n])))
        off += n
    print(f"{preset} S={S}: (tensor, ours vs fp64, reference fp32 vs fp64)", rows)
    for i, ours, ref in rows:
        assert ours <= max(3 * ref, 1e-4), (i, ours, ref)
    assert off == g64.size
