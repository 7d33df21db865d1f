"""bench.hpp harness on the B200 operators: run_op_bench (device-resident and
host drop-in) and the 100-config verify_sweep against the direct oracle with
the reference CLI's f32 tolerances (fftconv_cli.cpp:101-104)."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import LayerConfig, harness

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("resident", [True, False])
def test_run_op_bench(dev, resident):
    cfg = LayerConfig(5, 32, 16, 16, 8)
    rows = [harness.run_op_bench(cfg, op, iters=3, warmup=1, resident=resident) for op in harness.BenchOp]
    x, w, gy = harness.make_inputs(cfg, 1234)
    want = [oracle.forward_direct(x.astype(np.float64), w.astype(np.float64)).sum(),
            oracle.grad_input_direct(gy.astype(np.float64), w.astype(np.float64)).sum(),
            oracle.grad_weight_direct(gy.astype(np.float64), x.astype(np.float64)).sum()]
    for r, ref in zip(rows, want):
        assert r.stats.min_ms > 0 and r.stats.min_ms <= r.stats.mean_ms
        assert abs(r.checksum - ref) <= 1e-4 * max(1.0, abs(ref)) + 1e-3
    skipped = harness.run_op_bench(cfg, harness.BenchOp.gradinput, first_layer=True)
    assert skipped.skipped
    assert harness.bench_table(rows + [skipped]).count("\n") == 6


def test_verify_sweep_100_configs(dev):
    cfgs = harness.random_verify_configs(100, 2024)
    fns = {"forward": oracle.forward_direct, "grad_input": oracle.grad_input_direct,
           "grad_weight": oracle.grad_weight_direct}
    res = harness.verify_sweep(cfgs, 1234, lambda op, a, b: fns[op](a.astype(np.float64), b.astype(np.float64)))
    assert res.configs == 100
    assert res.within(1e-4, 1e-4, 1e-3), res
