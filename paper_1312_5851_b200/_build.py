"""In-tree build of every native artefact (nvcc cross-compiles sm_100a; no GPU needed).

* lib/libfftconv_b200.so        the product: K1/K3/K4 kernels + C ABI
* oracle/liboracle.so           test-only C restatement of the reference
* oracle/_ref/libfftconv_ref.so test/baseline-only build of the reference
                                (only where /root/reference exists)
* tests/cpp/dropin_test         C++ drop-in parity test against the
                                reference Tensor4/Weights4 types (only where
                                /root/reference exists; ships prebuilt)

Run: ``python -m paper_1312_5851_b200._build [--force]``.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libfftconv_b200.so")
REF_INCLUDE = os.environ.get("FFTCONV_REF_INCLUDE", "/root/reference/proj/include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "550",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd, **kw):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, **kw)


def build_cuda(force=False, verbose=False):
    sources = glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "fftconv_b200.h")]
    if not force and not _stale(LIB, sources):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cmd = [_nvcc()] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + [
        "-o", LIB, os.path.join(CSRC, "fftconv_b200.cu")]
    _run(cmd)
    return LIB


def build_oracle(force=False):
    args = ["make", "-C", os.path.join(ROOT, "oracle")]
    if force:
        args.append("-B")
    _run(args + ["oracle"])
    if os.path.isdir(os.path.join(REF_INCLUDE, "fftconv")):
        ref_so = os.path.join(ROOT, "oracle", "_ref", "libfftconv_ref.so")
        if force or _stale(ref_so, [os.path.join(ROOT, "oracle", "ref_shim.cpp")]):
            _run(args + ["ref", f"REF_INCLUDE={REF_INCLUDE}"])


def build_dropin_test(force=False):
    """C++ drop-in test: reference Tensor4/Weights4 + our header-only wrapper."""
    src = os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "dropin_test")
    if not os.path.exists(src) or not os.path.isdir(os.path.join(REF_INCLUDE, "fftconv")):
        return None
    deps = [src, os.path.join(ROOT, "include", "fftconv_b200.h"),
            os.path.join(ROOT, "include", "fftconv_b200", "conv_workspace.hpp")]
    if not force and not _stale(out, deps):
        return out
    _run(["g++", "-std=c++20", "-O2", "-pthread", f"-I{REF_INCLUDE}", f"-I{os.path.join(ROOT, 'include')}",
          "-o", out, src, f"-L{os.path.dirname(LIB)}", "-lfftconv_b200",
          "-Wl,-rpath,$ORIGIN/../../paper_1312_5851_b200/lib"])
    return out


def build(force=False, verbose=False):
    build_cuda(force, verbose)
    build_oracle(force)
    build_dropin_test(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
