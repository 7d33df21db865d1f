"""Runs the C++ drop-in test (tests/cpp/dropin_test.cpp): the reference's own
ConvWorkspace test cases on fftconv::b200::ConvWorkspace through the C ABI,
with the reference's fp64 direct convolution as the oracle and the
reference's exception classes checked.  The binary is built where the
reference headers exist and ships prebuilt to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "dropin_test")


def test_cpp_dropin_matches_reference_contract():
    if not os.path.exists(BIN):
        pytest.skip("dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
