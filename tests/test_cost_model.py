"""Cost model mirror (cost_model.hpp) against the reference, and the B200
roofline floors used by bench.py."""
import math

import pytest

import oracle
from paper_1312_5851_b200 import LayerConfig, cost_model as cm

CFGS = [(7, 32, 96, 96, 128), (11, 64, 256, 256, 128), (5, 32, 16, 16, 8), (3, 13, 5, 7, 2), (1, 1, 1, 1, 1)]


@pytest.mark.skipif(not oracle.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("cfg", CFGS)
@pytest.mark.parametrize("op", [0, 1, 2])
def test_op_counts_match_reference(cfg, op):
    ref = oracle.ref_cost_model(*cfg, 2.5, op)
    fn = (cm.ops_forward, cm.ops_grad_input, cm.ops_grad_weight)[op]
    got = fn(cm.CostParams(LayerConfig(*cfg), 2.5))
    for a, b in zip((got.direct_ops, got.transform_ops, got.pointwise_ops, got.inverse_ops), ref[:4]):
        assert math.isclose(a, b, rel_tol=1e-12, abs_tol=0)
    assert cm.memory_bytes(LayerConfig(*cfg)) == int(ref[4])
    assert cm.packed_memory_bytes(LayerConfig(*cfg), 4) == int(ref[5])


def test_ram_table_rows():
    # the first four rows follow the paper's table: 76 / 294 / 784 / 1159 MB
    assert [r[5] for r in cm.ram_table()[:4]] == [76, 294, 784, 1159]


def test_crossover_pad_pow2():
    rows = cm.crossover_table(96, 96, 128, 7, 2.5, [24, 32], pad_pow2=True)
    assert rows[0].fft_ops == cm.ops_forward(cm.CostParams(LayerConfig(7, 32, 96, 96, 128))).fft_ops()
    assert rows[1].direct_ops > 0


def test_roofline_floors_paper_point():
    c = LayerConfig(7, 32, 96, 96, 128)
    fl = cm.pass_floor_us(c, "forward", 6551.0, cm.gemm_tensor_tflops(1645.5, "f16x3"))
    assert math.isclose(sum(cm.kernel_bytes(c, "forward").values()), c.transform_bytes("forward"))
    # GEMM: 5.13 GFLOP at 548 TF/s = 9.4 us < 147 MB at 6551 GB/s = 22.4 us (HBM-bound)
    assert cm.gemm_bytes(c) == 8 * 544 * (128 * 96 * 2 + 96 * 96)
    assert 9 < fl["gemm_tensor"] < 10 and 22 < fl["gemm_hbm"] < 23 and fl["gemm"] == fl["gemm_hbm"]
    assert 20 < fl["r2c"] < 25 and 12 < fl["c2r"] < 15
    assert math.isclose(fl["pass"], fl["r2c"] + fl["gemm"] + fl["c2r"])
    rep = cm.roofline_report(c, {"forward": {"r2c": 41.0, "gemm": 31.0, "c2r": 27.0}}, 6551.0, 548.5)
    assert 0.5 < rep["forward"]["r2c_frac"] < 0.6 and 0.55 < rep["forward"]["pass_frac"] < 0.65


def test_gemm_tensor_rates():
    assert math.isclose(cm.gemm_tensor_tflops(1645.5, "f16x3"), 548.5)
    assert math.isclose(cm.gemm_tensor_tflops(1645.5, "tf32x3"), 274.25)
    # the wide layer's GEMM is tensor-heavier but still byte-bound at fp16x3
    w = LayerConfig(11, 64, 256, 256, 128)
    fl = cm.pass_floor_us(w, "forward", 6551.0, 548.5)
    assert fl["gemm_hbm"] > fl["gemm_tensor"]
    assert cm.pass_floor_us(w, "forward", 6551.0, 274.25)["gemm_tensor"] > fl["gemm_hbm"]
