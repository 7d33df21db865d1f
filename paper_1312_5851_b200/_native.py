"""ctypes binding of the C ABI in include/fftconv_b200.h.

The CUDA library is built in-tree (``paper_1312_5851_b200/lib``) by
``build.py``.  There is no fallback of any kind: if the library is missing or
cannot be loaded, every operator raises.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

HERE = os.path.dirname(os.path.abspath(__file__))
# FFTCONV_B200_LIB: alternative in-tree build for A/B kernel experiments.
LIB_PATH = os.environ.get("FFTCONV_B200_LIB") or os.path.join(HERE, "lib", "libfftconv_b200.so")

_sz = C.c_size_t
_p = C.c_void_p
_i = C.c_int

# Every symbol the header declares: (name, restype, argtypes).
SIGNATURES = [
    ("fftconv_b200_ws_create", _i, [_p, _sz, _i, C.POINTER(_p)]),
    ("fftconv_b200_ws_destroy", None, [_p]),
    ("fftconv_b200_last_error", C.c_char_p, [_p]),
    ("fftconv_b200_ws_info", _i, [_p, _p]),
    ("fftconv_b200_counters", _i, [_p, _p]),
    ("fftconv_b200_reset_counters", _i, [_p]),
    ("fftconv_b200_forward", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_forward_relu", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_grad_input", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_grad_weight", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_forward_fit", _i, [_p, _p, _sz, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, C.c_uint, _p]),
    ("fftconv_b200_grad_input_fit", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, _sz, _p]),
    ("fftconv_b200_grad_weight_fit", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_nccl_get_unique_id", _i, [_p]),
    ("fftconv_b200_nccl_comm_create", _i, [_p, _i, _i, _i, C.POINTER(_p)]),
    ("fftconv_b200_nccl_comm_destroy", _i, [_p]),
    ("fftconv_b200_grad_weight_sharded", _i,
     [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _p, _p, _i, C.c_uint, _p]),
    ("fftconv_b200_comm_wait", _i, [_p, _p]),
    ("fftconv_b200_grad_weight_sharded_host", _i,
     [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _p, _p, C.c_uint]),
    ("fftconv_b200_comm_ms", _i, [_p, _p]),
    ("fftconv_b200_forward_host", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, C.c_uint]),
    ("fftconv_b200_grad_input_host", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, C.c_uint]),
    ("fftconv_b200_grad_weight_host", _i, [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _p, C.c_uint]),
    ("fftconv_b200_spectrum_scratch_bytes", _sz, [_sz, _sz]),
    ("fftconv_b200_fft_2d_real_batch", _i, [_p, _sz, _sz, _p, _p, _sz, _p]),
    ("fftconv_b200_ifft_2d_real_batch", _i, [_p, _sz, _sz, _p, _p, _sz, _p]),
    ("fftconv_b200_set_stage_timing", _i, [_p, _i]),
    ("fftconv_b200_stage_ms", _i, [_p, _p]),
    ("fftconv_b200_last_launch_count", _i, [_p]),
    ("fftconv_b200_set_span_timing", _i, [_p, _i]),
    ("fftconv_b200_span_ms", _i, [_p, _p, _i]),
    ("fftconv_b200_relu_forward", _i, [_p, _p, _sz, _p]),
    ("fftconv_b200_relu_backward", _i, [_p, _p, _p, _sz, _p]),
    ("fftconv_b200_maxpool_forward", _i, [_p, _sz, _sz, _sz, _p, _p, _p]),
    ("fftconv_b200_maxpool_backward", _i, [_p, _p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_maxpool_relu_backward", _i, [_p, _p, _p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_fit_to", _i, [_p, _sz, _sz, _sz, _p, _sz, _p]),
    ("fftconv_b200_set_gemm_kind", _i, [_i]),
    ("fftconv_b200_ws_set_gemm_kind", _i, [_p, _i]),
    ("fftconv_b200_last_gemm_path", _i, [_p]),
    ("fftconv_b200_debug_r2c", _i, [_p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_debug_c2r", _i, [_p, _sz, _sz, _sz, _p, _p]),
    ("fftconv_b200_debug_cgemm", _i, [_p, _p, _p, _sz, _sz, _sz, _sz, _i, _p]),
]


class Layer(C.Structure):
    """fftconv_b200_layer == fftconv::LayerConfig {k, n, f, f', S}."""

    _fields_ = [("kernel", _sz), ("image", _sz), ("in_maps", _sz), ("out_maps", _sz), ("batch", _sz)]


class NativeLibraryMissing(ImportError):
    pass


@lru_cache(maxsize=None)
def lib() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} not found: build the CUDA library with `python build.py` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        # a symbol an older build (FFTCONV_B200_LIB A/B runs) lacks stays
        # unbound and fails loudly when called; the in-tree build exports
        # them all (tests/test_native_exports.py)
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.restype = res
        fn.argtypes = args
    return L


def last_error(ws=None) -> str:
    msg = lib().fftconv_b200_last_error(ws)
    return msg.decode() if msg else ""


GEMM_KINDS = {"f16x3": 0, "tf32x3": 1, "auto": 2}


def gemm_kind() -> str:
    """The K3 precision scheme in effect (include/fftconv_b200.h)."""
    prev = lib().fftconv_b200_set_gemm_kind(0)
    lib().fftconv_b200_set_gemm_kind(prev)
    return {v: k for k, v in GEMM_KINDS.items()}[prev]


def set_gemm_kind(kind: str) -> str:
    """Selects fp16x3 or 3xTF32 for K3; returns the previous kind."""
    prev = lib().fftconv_b200_set_gemm_kind(GEMM_KINDS[kind])
    return {v: k for k, v in GEMM_KINDS.items()}[prev]
