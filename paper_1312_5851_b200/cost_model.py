"""Cost model and roofline reporter.

Part 1 mirrors the reference's analytic model
(/root/reference/proj/include/fftconv/cost_model.hpp:10-172): operation
counts of the direct and FFT methods per training operation, the paper's
frequency-domain footprint and the packed footprint the implementation
allocates, the direct-vs-FFT crossover table and the RAM table.

Part 2 is the B200 roofline side used by bench.py: algorithmic HBM bytes of
the transform kernels and useful contraction flops per pass (SURVEY.md
section 8(d)), the floors they imply at measured peaks, and the fraction of
those floors a measured stage time reaches.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Sequence

from .errors import ConfigError
from .layer_config import LayerConfig, is_pow2, next_pow2

# ------------------------------------------------------------ reference model


@dataclass
class CostParams:  # cost_model.hpp:13-16
    config: LayerConfig
    C: float = 2.5


@dataclass
class OpCounts:  # cost_model.hpp:20-27
    direct_ops: float = 0.0
    transform_ops: float = 0.0
    pointwise_ops: float = 0.0
    inverse_ops: float = 0.0

    def fft_ops(self) -> float:
        return self.transform_ops + self.pointwise_ops + self.inverse_ops


def _xform_cost(C: float, n: float) -> float:  # cost_model.hpp:31-33
    return 0.0 if n <= 1 else 2.0 * C * n * n * math.log2(n)


def _dims(p: CostParams):
    c = p.config
    c.validate()
    return c.batch, c.in_maps, c.out_maps, c.image, c.kernel, c.output_size()


def ops_forward(p: CostParams) -> OpCounts:  # cost_model.hpp:39-53
    S, f, fp, n, k, no = _dims(p)
    t = _xform_cost(p.C, n)
    return OpCounts(S * fp * f * no * no * k * k, t * (S * f + fp * f), 4.0 * S * fp * f * n * n, t * (S * fp))


def ops_grad_input(p: CostParams) -> OpCounts:  # cost_model.hpp:57-71
    S, f, fp, n, k, no = _dims(p)
    t = _xform_cost(p.C, no)
    return OpCounts(S * fp * f * n * n * k * k, t * (S * fp + fp * f), 4.0 * S * fp * f * no * no, t * (S * f))


def ops_grad_weight(p: CostParams) -> OpCounts:  # cost_model.hpp:75-89
    S, f, fp, n, k, no = _dims(p)
    t = _xform_cost(p.C, n)
    return OpCounts(S * fp * f * k * k * no * no, t * (S * fp + S * f), 4.0 * S * fp * f * n * n, t * (fp * f))


def memory_bytes(c: LayerConfig) -> int:  # cost_model.hpp:93-99
    c.validate()
    return 4 * c.image * (c.image + 1) * (c.batch * c.in_maps + c.batch * c.out_maps + c.in_maps * c.out_maps)


def packed_memory_bytes(c: LayerConfig, scalar_bytes: int) -> int:  # cost_model.hpp:103-110
    c.validate()
    return (c.batch * c.in_maps + c.batch * c.out_maps + c.in_maps * c.out_maps) * c.bins() * 2 * scalar_bytes


@dataclass
class CrossoverRow:  # cost_model.hpp:116-120
    image: int
    direct_ops: float
    fft_ops: float


def crossover_table(f: int, fp: int, S: int, k: int, C: float, n_values: Sequence[int],
                    pad_pow2: bool = False) -> List[CrossoverRow]:  # cost_model.hpp:124-146
    if not n_values:
        raise ConfigError("crossover table: at least one image size required")
    rows = []
    for n in n_values:
        at_n = ops_forward(CostParams(LayerConfig(k, n, f, fp, S), C))
        fft = at_n.fft_ops()
        if pad_pow2 and not is_pow2(n):
            fft = ops_forward(CostParams(LayerConfig(k, next_pow2(n), f, fp, S), C)).fft_ops()
        rows.append(CrossoverRow(n, at_n.direct_ops, fft))
    return rows


RAM_CONFIGS = [(128, 16, 96, 256), (128, 32, 96, 256), (64, 64, 96, 256), (128, 64, 96, 256),
               (128, 16, 256, 384), (128, 32, 256, 384), (128, 16, 384, 384), (128, 32, 384, 384)]


def ram_table():  # cost_model.hpp:156-170: (S, n, f, f', bytes, decimal MB)
    out = []
    for S, n, f, fp in RAM_CONFIGS:
        b = memory_bytes(LayerConfig(1, n, f, fp, S))
        out.append((S, n, f, fp, b, int(round(b / 1e6))))
    return out


# ------------------------------------------------------------ B200 roofline

OPS = ("forward", "grad_input", "grad_weight")


def kernel_bytes(c: LayerConfig, op: str) -> Dict[str, int]:
    """Algorithmic HBM bytes per launch of the transform kernels of one pass:
    K1 reads every real input plane once and writes its half spectrum once
    (both operands, one launch); K4 reads the product spectrum once and
    writes only the cropped output."""
    S, f, fo, n, k = c.batch, c.in_maps, c.out_maps, c.image, c.kernel
    no, bins = c.output_size(), c.bins()
    if op == "forward":
        return {"r2c": 4 * (S * f * n * n + fo * f * k * k) + 8 * bins * (S * f + fo * f),
                "c2r": 8 * bins * S * fo + 4 * S * fo * no * no}
    if op == "grad_input":
        return {"r2c": 4 * (S * fo * no * no + fo * f * k * k) + 8 * bins * (S * fo + fo * f),
                "c2r": 8 * bins * S * f + 4 * S * f * n * n}
    if op == "grad_weight":
        return {"r2c": 4 * (S * f * n * n + S * fo * no * no) + 8 * bins * (S * f + S * fo),
                "c2r": 8 * bins * fo * f + 4 * fo * f * k * k}
    raise ValueError(op)


def gemm_bytes(c: LayerConfig) -> int:
    """Algorithmic HBM bytes of the per-bin GEMM (any op): both operand
    spectra read once, the product spectrum written once.  The three ops
    pair the dims (S, f), (f', f), (S, f') in some order."""
    S, f, fo, bins = c.batch, c.in_maps, c.out_maps, c.bins()
    return 8 * bins * (S * f + fo * f + S * fo)


def gemm_tensor_tflops(bf16_tflops: float, kind: str = "f16x3") -> float:
    """Useful complex-GEMM rate of the tensor cores: 3 MMA passes per
    product, at the fp16 (= bf16) rate for fp16x3 or half of it for 3xTF32."""
    return bf16_tflops / 3.0 if kind == "f16x3" else bf16_tflops / 2.0 / 3.0


def pass_floor_us(c: LayerConfig, op: str, hbm_gbs: float, tensor_tflops: float) -> Dict[str, float]:
    """Floors of one pass at the given peaks: transform bytes / HBM, and for
    the GEMM the larger of contraction flops / tensor peak and its operand +
    product bytes / HBM (pass-level roofline), in
    microseconds."""
    kb = kernel_bytes(c, op)
    out = {k: v / (hbm_gbs * 1e9) * 1e6 for k, v in kb.items()}
    out["gemm_tensor"] = c.contraction_flops() / (tensor_tflops * 1e12) * 1e6
    out["gemm_hbm"] = gemm_bytes(c) / (hbm_gbs * 1e9) * 1e6
    out["gemm"] = max(out["gemm_tensor"], out["gemm_hbm"])
    out["pass"] = out["r2c"] + out["gemm"] + out["c2r"]
    return out


def roofline_report(c: LayerConfig, stage_us: Dict[str, Dict[str, float]], hbm_gbs: float,
                    tensor_tflops: float) -> Dict[str, Dict[str, float]]:
    """stage_us[op] = {"r2c": t, "gemm": t, "c2r": t} measured (us) ->
    per stage: floor, measured, fraction of the floor reached; per pass:
    the fusion-proof pass-level fraction (sum of floors / measured pass)."""
    rep = {}
    for op, st in stage_us.items():
        fl = pass_floor_us(c, op, hbm_gbs, tensor_tflops)
        r = {f"{k}_floor_us": fl[k] for k in ("r2c", "gemm", "c2r")}
        for k in ("r2c", "gemm", "c2r"):
            if k in st and st[k] > 0:
                r[f"{k}_us"] = st[k]
                r[f"{k}_frac"] = fl[k] / st[k]
        tot = sum(st.get(k, 0.0) for k in ("r2c", "gemm", "c2r"))
        if tot > 0:
            r["pass_us"] = tot
            r["pass_frac"] = fl["pass"] / tot
        rep[op] = r
    return rep
