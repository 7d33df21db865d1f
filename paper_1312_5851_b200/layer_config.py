"""LayerConfig and power-of-two helpers (/root/reference/proj/include/fftconv/layer_config.hpp:11-40)."""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError


def next_pow2(n: int) -> int:
    """layer_config.hpp:11-15"""
    m = 1
    while m < n:
        m <<= 1
    return m


def is_pow2(n: int) -> bool:
    """layer_config.hpp:17"""
    return n != 0 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class LayerConfig:
    """One conv layer shape {k, n, f, f', S} (layer_config.hpp:22-40)."""

    kernel: int  # k
    image: int  # n
    in_maps: int  # f
    out_maps: int  # f'
    batch: int  # S

    def output_size(self) -> int:
        """n' = n - k + 1 (layer_config.hpp:29)."""
        return self.image - self.kernel + 1

    def fft_size(self) -> int:
        """m = next_pow2(n) (layer_config.hpp:30)."""
        return next_pow2(self.image)

    def bins(self) -> int:
        m = self.fft_size()
        return m * (m // 2 + 1)

    def validate(self) -> None:
        """layer_config.hpp:32-39"""
        if min(self.kernel, self.image, self.in_maps, self.out_maps, self.batch) <= 0:
            raise ConfigError("layer config: all parameters must be >= 1")
        if self.kernel > self.image:
            raise ConfigError(f"layer config: kernel {self.kernel} exceeds image {self.image}")

    def as_tuple(self):
        return (self.kernel, self.image, self.in_maps, self.out_maps, self.batch)

    # -- analytic figures used by the bench/roofline
    def equiv_flops(self) -> int:
        """Direct-convolution-equivalent FLOPs per pass: 2*S*f*f'*n'^2*k^2."""
        no = self.output_size()
        return 2 * self.batch * self.in_maps * self.out_maps * no * no * self.kernel * self.kernel

    def contraction_flops(self) -> int:
        """Useful complex-GEMM FLOPs per pass: 8*bins*S*f*f'."""
        return 8 * self.bins() * self.batch * self.in_maps * self.out_maps

    def transform_bytes(self, op: str) -> int:
        """Minimal HBM bytes of the transform stages of one pass."""
        S, f, fo, n, k = self.batch, self.in_maps, self.out_maps, self.image, self.kernel
        no, bins = self.output_size(), self.bins()
        if op == "forward":
            return 4 * (S * f * n * n + fo * f * k * k) + 8 * bins * (S * f + fo * f) + 8 * bins * S * fo + 4 * S * fo * no * no
        if op == "grad_input":
            return 4 * (S * fo * no * no + fo * f * k * k) + 8 * bins * (S * fo + fo * f) + 8 * bins * S * f + 4 * S * f * n * n
        if op == "grad_weight":
            return 4 * (S * f * n * n + S * fo * no * no) + 8 * bins * (S * f + S * fo) + 8 * bins * fo * f + 4 * fo * f * k * k
        raise ValueError(op)
