import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def dev():
    import torch

    return torch.device("cuda:0")


@pytest.fixture(params=["f16x3", "tf32x3", "auto"])
def gemm_kind(request):
    """Runs the test under each K3 precision scheme (fftconv_b200_set_gemm_kind)."""
    from paper_1312_5851_b200 import _native

    kind = {"f16x3": 0, "tf32x3": 1, "auto": 2}[request.param]
    prev = _native.lib().fftconv_b200_set_gemm_kind(kind)
    yield request.param
    _native.lib().fftconv_b200_set_gemm_kind(prev)
