"""Public packed-spectrum API of the reference (fft.hpp:105-152, :209-243) on
the B200 transform kernels: ``HalfSpectrum``, ``fft_2d_real_batch`` and
``ifft_2d_real_batch``.  SURVEY.md section 8(a) row a14: not used by the
operators themselves, but the reference's unit-level surface for K1/K4
(fft_test.cpp:122-199).

Packing is the reference's: per plane m rows x (m/2 + 1) packed columns,
``full[u][v] = conj(full[(m-u)%m][(m-v)%m])`` for the unstored columns.  The
kernels' internal half spectrum keeps the other half (rows u <= m/2, all
columns v), so these wrappers repack at the boundary through the same
Hermitian identity; they are convenience / parity entry points, not a hot
path.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import SizeError
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


def fft_2d_real_batch(t, m: int | None = None) -> HalfSpectrum:
    """fft.hpp:209-225: packed forward transform of every (batch, map) plane
    of t [batch][maps][m][m] (fp32; CUDA tensor or host array).  Planes must
    already be padded to the plan size m (``size_error`` otherwise)."""
    torch = _torch()
    from . import kernels

    t = torch.as_tensor(t, dtype=torch.float32)
    if t.device.type != "cuda":
        t = t.cuda()
    B, F, R, Cc = t.shape
    m = R if m is None else m
    if m == 0 or not is_pow2(m):
        raise SizeError("fft_2d_real_batch: plan size must be a power of two")
    if R != m or Cc != m:
        raise SizeError("fft_2d_real_batch: planes must be padded to the plan size")
    ours = kernels.r2c(t.reshape(B * F, m, m), m)  # [P][m/2+1][m]: half over rows
    return HalfSpectrum(_rows_to_cols(ours, m).reshape(B, F, m, m // 2 + 1))


def ifft_2d_real_batch(s: HalfSpectrum, m: int | None = None):
    """fft.hpp:227-243: inverse of fft_2d_real_batch, full real m x m planes
    (scaled by 1/m^2 like the reference's two 1/m passes)."""
    from . import kernels

    B, F, R, pc = s.data.shape
    m = R if m is None else m
    if R != m:
        raise SizeError("ifft_2d_real_batch: spectrum rows do not match plan size")
    ours = _cols_to_rows(s.data.reshape(B * F, m, pc), m)  # [P][m/2+1][m]
    return kernels.c2r(ours, m).reshape(B, F, m, m)


def _rows_to_cols(h, m: int):
    """[P][m/2+1][m] (u <= m/2, all v) -> [P][m][m/2+1] (all u, v <= m/2):
    F[u][v] = conj(F[m-u][(m-v) % m]) for u > m/2."""
    torch = _torch()
    pc = m // 2 + 1
    u = torch.arange(m, device=h.device).view(m, 1)
    v = torch.arange(pc, device=h.device).view(1, pc)
    low = u <= m // 2
    ru = torch.where(low, u, m - u).expand(m, pc)
    rv = torch.where(low, v, (m - v) % m).expand(m, pc)
    out = h[:, ru, rv]
    return torch.where(low.expand(m, pc), out, out.conj())


def _cols_to_rows(c, m: int):
    """[P][m][m/2+1] (all u, v <= m/2) -> [P][m/2+1][m] (u <= m/2, all v):
    F[u][v] = conj(F[(m-u) % m][m-v]) for v > m/2."""
    torch = _torch()
    pc = m // 2 + 1
    u = torch.arange(pc, device=c.device).view(pc, 1)
    v = torch.arange(m, device=c.device).view(1, m)
    low = v <= m // 2
    ru = torch.where(low, u, (m - u) % m).expand(pc, m)
    rv = torch.where(low, v, m - v).expand(pc, m)
    out = c[:, ru, rv]
    return torch.where(low.expand(pc, m), out, out.conj()).contiguous()
