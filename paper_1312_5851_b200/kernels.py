"""Unit-level entry points to the individual kernels (K1 r2c, K4 c2r, K3
per-bin complex GEMM) for parity tests.  CUDA tensors only."""
from __future__ import annotations

import ctypes as C

from . import _native
from .errors import raise_for_status


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream(t):
    import torch

    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def r2c(planes, m: int):
    """[P][src][src] fp32 -> [P][m/2+1][m] complex64 (half over rows u, all v)."""
    import torch

    planes = planes.contiguous()
    P, src, _ = planes.shape
    out = torch.empty((P, m // 2 + 1, m, 2), dtype=torch.float32, device=planes.device)
    code = _native.lib().fftconv_b200_debug_r2c(_ptr(planes), P, src, m, _ptr(out), _stream(planes))
    raise_for_status(code, _native.last_error(None))
    return torch.view_as_complex(out)


def c2r(spec, crop: int):
    """[P][m/2+1][m] complex64 -> [P][crop][crop] fp32 (scaled by 1/m^2)."""
    import torch

    P, pc, m = spec.shape
    s = torch.view_as_real(spec.contiguous()).contiguous()
    out = torch.empty((P, crop, crop), dtype=torch.float32, device=spec.device)
    code = _native.lib().fftconv_b200_debug_c2r(_ptr(s), P, m, crop, _ptr(out), _stream(s))
    raise_for_status(code, _native.last_error(None))
    return out


def cgemm(a, b, mode: int):
    """Per-bin complex GEMM: a [bins][M][K], b [bins][N][K] complex64 -> out [bins][N][M].
    mode 0: sum_k a conj(b); 1: sum_k a b; 2: sum_k conj(a) b."""
    import torch

    bins, M, K = a.shape
    _, N, _ = b.shape
    ar = torch.view_as_real(a.contiguous()).contiguous()
    br = torch.view_as_real(b.contiguous()).contiguous()
    out = torch.empty((bins, N, M, 2), dtype=torch.float32, device=a.device)
    code = _native.lib().fftconv_b200_debug_cgemm(_ptr(ar), _ptr(br), _ptr(out), bins, M, N, K, int(mode),
                                                  _stream(ar))
    raise_for_status(code, _native.last_error(None))
    return torch.view_as_complex(out)
