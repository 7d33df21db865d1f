"""Harness mirror of bench.hpp (CPU): summarize_ms, random_verify_configs
and the CLI report schema, checked against the reference where it is built."""
import math

import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import LayerConfig, harness


def test_summarize_ms():
    s = harness.summarize_ms([3.0, 1.0, 2.0, 10.0])
    assert (s.mean_ms, s.min_ms, s.median_ms) == (4.0, 1.0, 2.5)
    assert math.isclose(s.std_ms, np.std([3, 1, 2, 10], ddof=1))
    assert harness.summarize_ms([5.0]).std_ms == 0.0


def test_random_verify_configs_match_reference_draws():
    got = [(c.kernel, c.image, c.in_maps, c.out_maps, c.batch) for c in harness.random_verify_configs(100, 2024)]
    assert got == [tuple(c) for c in oracle.random_verify_configs(100, 2024)]
    for k, n, f, fo, S in got:
        assert 1 <= k <= min(11, n) and 2 <= n <= 32 and 1 <= f <= 8 and 1 <= fo <= 8 and 1 <= S <= 4


def test_bench_table_schema():
    cfg = LayerConfig(5, 32, 16, 16, 8)
    rows = [harness.BenchResult(harness.BenchOp.output, "b200", cfg, 10, 3, 1, 1234,
                                harness.BenchStats(1.0, 0.1, 0.9, 1.0), 12.5),
            harness.BenchResult(harness.BenchOp.gradinput, "b200", cfg, 10, 3, 1, 1234, skipped=True)]
    csv = harness.bench_table(rows, "csv").splitlines()
    assert csv[0] == "op,method,k,n,f,fprime,S,iters,threads,seed,mean_ms,std_ms,min_ms,checksum"
    assert csv[1].startswith("updateOutput,b200,5,32,16,16,8,10,1,1234,1.000,0.100,0.900,12.5")
    assert csv[2] == "updateGradInput,b200,5,32,16,16,8,10,1,1234,,,,"
    assert csv[3].startswith("total,b200,")
    md = harness.bench_table(rows, "md").splitlines()
    assert md[0].split("|")[1].strip() == "op" and "skipped" in md[3]
