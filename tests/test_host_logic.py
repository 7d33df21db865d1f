"""Host-side logic that needs no GPU: layer maths, roofline formulas,
generator parity, error taxonomy, sharding arithmetic, bench helpers."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import (CapacityError, ConfigError, CudaError, FftconvError, LayerConfig, PlanError,
                                  ShapeError, SizeError, is_pow2, next_pow2)
from paper_1312_5851_b200.errors import raise_for_status
from paper_1312_5851_b200.rng import fill_uniform, splitmix64
from paper_1312_5851_b200.sharded import shard_range

P = LayerConfig(7, 32, 96, 96, 128)
W = LayerConfig(11, 64, 256, 256, 128)
C = LayerConfig(5, 32, 16, 16, 8)


def test_pow2_helpers():
    assert [next_pow2(n) for n in (1, 2, 3, 7, 9, 32, 33)] == [1, 2, 4, 8, 16, 32, 64]
    assert is_pow2(64) and not is_pow2(6) and not is_pow2(0)


def test_layer_config():
    assert P.output_size() == 26 and P.fft_size() == 32 and P.bins() == 544
    assert W.output_size() == 54 and W.bins() == 2112
    with pytest.raises(ConfigError):
        LayerConfig(0, 8, 1, 1, 1).validate()
    with pytest.raises(ConfigError):
        LayerConfig(9, 8, 1, 1, 1).validate()


def test_roofline_formulas_match_survey():
    """E = 78.15 / 5919.6 / 0.080 GFLOP; contraction 5.13 / 141.7
    GFLOP; transform bytes 232.4 MB (P) and 3.17 GB (W) per pass."""
    assert P.equiv_flops() / 1e9 == pytest.approx(78.15, rel=1e-3)
    assert W.equiv_flops() / 1e9 == pytest.approx(5919.6, rel=1e-3)
    assert C.equiv_flops() / 1e9 == pytest.approx(0.080, rel=2e-2)
    assert P.contraction_flops() / 1e9 == pytest.approx(5.13, rel=1e-3)
    assert W.contraction_flops() / 1e9 == pytest.approx(141.7, rel=1e-3)
    for op in ("forward", "grad_input", "grad_weight"):
        assert P.transform_bytes(op) / 1e6 == pytest.approx(232.4, rel=0.05)
        assert W.transform_bytes(op) / 1e9 == pytest.approx(3.17, rel=0.05)


def test_numpy_generator_is_the_reference_generator():
    a = fill_uniform((2, 3, 7, 7), 1234, 1)
    b = oracle.fill_uniform((2, 3, 7, 7), 1234, 1)
    assert np.array_equal(a, b)
    a64 = fill_uniform((50,), 99, 3, stream=2, dtype=np.float64)
    b64 = oracle.fill_uniform((50,), 99, 3, stream=2, dtype=np.float64)
    assert np.array_equal(a64, b64)
    assert splitmix64(0) == oracle.lib().orc_splitmix64(0)


def test_error_taxonomy():
    for code, cls in ((1, SizeError), (2, ShapeError), (3, ConfigError), (4, CapacityError), (5, PlanError),
                      (6, CudaError)):
        with pytest.raises(cls):
            raise_for_status(code, "x")
        assert issubclass(cls, FftconvError)
    raise_for_status(0, "")


@pytest.mark.parametrize("S,world", [(128, 1), (128, 2), (128, 8), (7, 3), (3, 4), (128, 6)])
def test_shard_range_partitions_the_batch(S, world):
    seen = []
    for r in range(world):
        b0, b1 = shard_range(S, world, r)
        assert b0 <= b1
        seen.extend(range(b0, b1))
    assert seen == list(range(S))
    sizes = [shard_range(S, world, r)[1] - shard_range(S, world, r)[0] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_bench_config_parsing():
    import bench

    cfg, label = bench.parse_config("paper")
    assert cfg == (7, 32, 96, 96, 128) and "paper" in label
    cfg, _ = bench.parse_config("sweep:64,13")
    assert cfg == (13, 64, 96, 96, 128)
    cfg, _ = bench.parse_config("wide")
    assert cfg == (11, 64, 256, 256, 128)


def test_fill_uniform_offset_is_a_slice():
    from paper_1312_5851_b200.rng import fill_uniform

    full = fill_uniform((4, 3, 5), 99, 1)
    assert np.array_equal(fill_uniform((2, 3, 5), 99, 1, offset=2 * 15), full[2:4])
