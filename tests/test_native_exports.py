"""The product library loads without a GPU, exports every symbol declared in
include/fftconv_b200.h, carries real sm_100a tcgen05/TMA code, and rejects
invalid configs before touching the device.  CPU only (no compute calls)."""
import os
import re
import subprocess

import pytest

from paper_1312_5851_b200 import ConfigError, ConvWorkspace, _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fftconv_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fftconv_b200_\w+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _native.lib()
    declared = header_functions()
    assert len(declared) >= 18
    for name in declared:
        assert hasattr(L, name), name
    bound = {s[0] for s in _native.SIGNATURES}
    assert bound == set(declared)


def test_library_is_sm100a_with_tcgen05_and_tma():
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    elf = subprocess.run([cuobjdump, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in elf
    sass = subprocess.run([cuobjdump, "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert re.search(r"UTC\w*MMA", sass), "no tcgen05.mma in SASS"
    assert "UTMALDG" in sass, "no TMA loads in SASS"
    assert "LDTM" in sass, "no tcgen05.ld in SASS"


def test_empty_and_invalid_configs_rejected_before_device_work():
    with pytest.raises(ConfigError):
        ConvWorkspace([], device=0)
    with pytest.raises(ConfigError):
        ConvWorkspace([(5, 3, 1, 1, 1)], device=0)  # kernel > image
    with pytest.raises(ConfigError):
        ConvWorkspace([(3, 8, 0, 1, 1)], device=0)


def test_last_error_message_mirrors_reference_text():
    with pytest.raises(ConfigError, match="at least one layer config required"):
        ConvWorkspace([], device=0)
