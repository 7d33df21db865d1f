"""Public packed-spectrum API of the reference (fft.hpp:105-152, :209-243) on
the B200 transform kernels: ``HalfSpectrum``, ``fft_2d_real_batch`` and
``ifft_2d_real_batch``.  SURVEY.md section 8(a) row a14: not used by the
operators themselves, but the reference's unit-level surface for K1/K4
(fft_test.cpp:122-199).

Packing is the reference's: per plane m rows x (m/2 + 1) packed columns,
``full[u][v] = conj(full[(m-u)%m][(m-v)%m])`` for the unstored columns.  The
kernels' internal half spectrum keeps the other half (rows u <= m/2, all
columns v); the C-ABI entry points (include/fftconv_b200.h,
fftconv_b200_fft_2d_real_batch / _ifft_) repack at the boundary with one
device kernel through the same Hermitian identity.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import PlanError, SizeError
from .layer_config import is_pow2


def _torch():
    import torch

    return torch


@dataclass
class HalfSpectrum:
    """fft.hpp:105-152: complex64 tensor [batch][maps][m][m/2 + 1] on the GPU."""

    data: object  # torch.complex64, CUDA

    @classmethod
    def zeros(cls, batch: int, maps: int, m: int, device="cuda"):
        if batch == 0 or maps == 0 or m == 0:
            raise SizeError("HalfSpectrum: all dimensions must be >= 1")
        torch = _torch()
        return cls(torch.zeros((batch, maps, m, m // 2 + 1), dtype=torch.complex64, device=device))

    def batch(self) -> int:
        return self.data.shape[0]

    def maps(self) -> int:
        return self.data.shape[1]

    def rows(self) -> int:
        return self.data.shape[2]

    def packed_cols(self) -> int:
        return self.data.shape[3]

    def plane_size(self) -> int:
        return self.rows() * self.packed_cols()

    def packed_bin(self, b: int, f: int, u: int, v: int) -> complex:
        return complex(self.data[b, f, u, v].item())

    def full_bin(self, b: int, f: int, u: int, v: int) -> complex:
        """Any bin of the full m x m spectrum (Hermitian unpacking, fft.hpp:140-144)."""
        if v < self.packed_cols():
            return self.packed_bin(b, f, u, v)
        m = self.rows()
        return self.packed_bin(b, f, (m - u) % m, m - v).conjugate()


def _call(fn, src, P, m, dst):
    import ctypes as C

    from . import _native
    from .errors import raise_for_status

    torch = _torch()
    L = _native.lib()
    nbytes = int(L.fftconv_b200_spectrum_scratch_bytes(P, m))
    scratch = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=src.device)
    code = fn(C.c_void_p(src.data_ptr()), P, m, C.c_void_p(dst.data_ptr()), C.c_void_p(scratch.data_ptr()), nbytes,
              C.c_void_p(torch.cuda.current_stream(src.device).cuda_stream))
    raise_for_status(code, _native.last_error(None))


def fft_2d_real_batch(t, m: int | None = None) -> HalfSpectrum:
    """fft.hpp:209-225: packed forward transform of every (batch, map) plane
    of t [batch][maps][m][m] (fp32; CUDA tensor or host array), through
    fftconv_b200_fft_2d_real_batch (K1 + a repack into the reference
    packing).  Planes must already be padded to the plan size m
    (``size_error`` otherwise)."""
    from . import _native

    torch = _torch()
    t = torch.as_tensor(t, dtype=torch.float32)
    if t.device.type != "cuda":
        t = t.cuda()
    t = t.contiguous()
    B, F, R, Cc = t.shape
    m = R if m is None else m
    if m == 0 or not is_pow2(m):
        raise PlanError(f"fft plan: size {m} is not a power of 2")
    if R != m or Cc != m:
        raise SizeError("fft_2d_real_batch: planes must be padded to the plan size")
    if B == 0 or F == 0:
        raise SizeError("HalfSpectrum: all dimensions must be >= 1")
    out = torch.empty((B, F, m, m // 2 + 1), dtype=torch.complex64, device=t.device)
    _call(_native.lib().fftconv_b200_fft_2d_real_batch, t, B * F, m, out)
    return HalfSpectrum(out)


def ifft_2d_real_batch(s: HalfSpectrum, m: int | None = None):
    """fft.hpp:227-243: inverse of fft_2d_real_batch, full real m x m planes
    (scaled by 1/m^2 like the reference's two 1/m passes), through
    fftconv_b200_ifft_2d_real_batch."""
    from . import _native

    torch = _torch()
    B, F, R, pc = s.data.shape
    m = R if m is None else m
    if m == 0 or not is_pow2(m):
        raise PlanError(f"fft plan: size {m} is not a power of 2")
    if R != m:
        raise SizeError("ifft_2d_real_batch: spectrum rows do not match plan size")
    spec = s.data.contiguous()
    out = torch.empty((B, F, m, m), dtype=torch.float32, device=spec.device)
    _call(_native.lib().fftconv_b200_ifft_2d_real_batch, spec, B * F, m, out)
    return out
