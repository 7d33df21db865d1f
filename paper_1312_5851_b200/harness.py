"""Benchmark / verification harness of the B200 operators in the reference's
own terms.

Mirrors /root/reference/proj/include/fftconv/bench.hpp:
  * BenchOp / method names (:17-31) and summarize_ms (:45-66);
  * run_op_bench (:72-145): inputs from the reference generator
    (fill_uniform, roles input / weights / grad_output), workspace built
    outside the clock, every transform inside it, checksum = sum of the
    output elements, first-layer updateGradInput skipped;
  * random_verify_configs (:164-183) and verify_sweep (:187-222), the
    sup-norm relative error of tensor.hpp:177-181;
and the report rows of the reference CLI (tools/fftconv_cli.cpp:144-200):
CSV columns op,method,k,n,f,fprime,S,iters,threads,seed,mean_ms,std_ms,
min_ms,checksum, or the markdown columns op,method,mean_ms,std_ms,min_ms,
median_ms,checksum, plus per-method totals.

The B200 method runs either with device-resident inputs (CUDA-event time
per call, `resident=True`) or through the host drop-in (wall time including
the copies, `resident=False`).  verify_sweep compares against a caller-supplied
reference (the direct oracle lives in tests/, not in the product).
"""
from __future__ import annotations

import enum
import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from .errors import ConfigError
from .layer_config import LayerConfig
from .rng import ROLE_GRAD_OUTPUT, ROLE_INPUT, ROLE_WEIGHTS, fill_uniform, splitmix64
from .workspace import ConvWorkspace


class BenchOp(enum.IntEnum):  # bench.hpp:17
    output = 0
    gradinput = 1
    gradweight = 2


OP_NAMES = {BenchOp.output: "updateOutput", BenchOp.gradinput: "updateGradInput",
            BenchOp.gradweight: "accGradParameters"}  # bench.hpp:20-27
METHOD = "b200"


@dataclass
class BenchStats:  # bench.hpp:33-35
    mean_ms: float = 0.0
    std_ms: float = 0.0
    min_ms: float = 0.0
    median_ms: float = 0.0


def summarize_ms(samples: Sequence[float]) -> BenchStats:
    """bench.hpp:45-66: mean, sample std (n-1), min, median."""
    s = BenchStats()
    if not samples:
        return s
    n = len(samples)
    s.mean_ms = sum(samples) / n
    s.min_ms = min(samples)
    if n > 1:
        s.std_ms = math.sqrt(sum((v - s.mean_ms) ** 2 for v in samples) / (n - 1))
    v = sorted(samples)
    s.median_ms = v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])
    return s


@dataclass
class BenchResult:  # bench.hpp:37-43
    op: BenchOp
    method: str
    config: LayerConfig
    iters: int
    warmup: int
    threads: int
    seed: int
    stats: BenchStats = field(default_factory=BenchStats)
    checksum: float = 0.0
    skipped: bool = False


def make_inputs(cfg: LayerConfig, seed: int):
    """x, w, gy exactly as run_op_bench fills them (bench.hpp:100-106)."""
    no = cfg.output_size()
    x = fill_uniform((cfg.batch, cfg.in_maps, cfg.image, cfg.image), seed, ROLE_INPUT)
    w = fill_uniform((cfg.out_maps, cfg.in_maps, cfg.kernel, cfg.kernel), seed, ROLE_WEIGHTS)
    gy = fill_uniform((cfg.batch, cfg.out_maps, no, no), seed, ROLE_GRAD_OUTPUT)
    return x, w, gy


def run_op_bench(cfg: LayerConfig, op: BenchOp, iters: int = 10, warmup: int = 3, seed: int = 1234,
                 first_layer: bool = False, resident: bool = True, device: int = 0) -> BenchResult:
    """bench.hpp:72-145 for the B200 operators."""
    cfg.validate()
    if iters < 1:
        raise ConfigError("bench: iters must be >= 1")
    r = BenchResult(BenchOp(op), METHOD, cfg, iters, warmup, 1, seed)
    if op == BenchOp.gradinput and first_layer:
        r.skipped = True
        return r
    x, w, gy = make_inputs(cfg, seed)
    ws = ConvWorkspace([cfg], device=device)
    if resident:
        import torch

        dev = torch.device("cuda", device)
        x, w, gy = (torch.from_numpy(a).to(dev) for a in (x, w, gy))
    call = {BenchOp.output: lambda: ws.forward(x, w), BenchOp.gradinput: lambda: ws.grad_input(gy, w),
            BenchOp.gradweight: lambda: ws.grad_weight(gy, x)}[BenchOp(op)]
    for _ in range(warmup):
        call()
    samples = []
    for _ in range(iters):
        if resident:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = call()
            e1.record()
            e1.synchronize()
            samples.append(e0.elapsed_time(e1))
            r.checksum = float(out.double().sum())
        else:
            t0 = time.perf_counter()
            out = call()
            samples.append((time.perf_counter() - t0) * 1e3)
            r.checksum = float(np.asarray(out, np.float64).sum())
    r.stats = summarize_ms(samples)
    return r


def bench_table(rows: List[BenchResult], fmt: str = "csv") -> str:
    """The reference CLI's report (fftconv_cli.cpp:144-200): one row per
    (op, method) plus a per-method total over the ops that ran."""
    md = fmt == "md"
    head = (["op", "method", "mean_ms", "std_ms", "min_ms", "median_ms", "checksum"] if md else
            ["op", "method", "k", "n", "f", "fprime", "S", "iters", "threads", "seed", "mean_ms", "std_ms",
             "min_ms", "checksum"])
    body = []

    def fmt_ms(v):
        return f"{v:.3f}"

    def fmt_val(v):
        return f"{v:.6g}"

    def cells(op_label, method, st, checksum, skipped, r0):
        if md:
            return [op_label, method] + (["skipped", "-", "-", "-", "-"] if skipped else
                                         [fmt_ms(st.mean_ms), fmt_ms(st.std_ms), fmt_ms(st.min_ms),
                                          fmt_ms(st.median_ms), fmt_val(checksum)])
        c = r0.config
        base = [op_label, method, str(c.kernel), str(c.image), str(c.in_maps), str(c.out_maps), str(c.batch),
                str(r0.iters), str(r0.threads), str(r0.seed)]
        return base + (["", "", "", ""] if skipped else
                       [fmt_ms(st.mean_ms), fmt_ms(st.std_ms), fmt_ms(st.min_ms), fmt_val(checksum)])

    for r in rows:
        body.append(cells(OP_NAMES[r.op], r.method, r.stats, r.checksum, r.skipped, r))
    for method in dict.fromkeys(r.method for r in rows):
        ran = [r for r in rows if r.method == method and not r.skipped]
        if not ran:
            continue
        tot = BenchStats(sum(r.stats.mean_ms for r in ran), math.sqrt(sum(r.stats.std_ms ** 2 for r in ran)),
                         sum(r.stats.min_ms for r in ran), sum(r.stats.median_ms for r in ran))
        body.append(cells("total", method, tot, sum(r.checksum for r in ran), False, ran[0]))
    if md:
        width = [max(len(h), *(len(b[i]) for b in body)) for i, h in enumerate(head)]
        line = lambda cs: "| " + " | ".join(c.ljust(w) for c, w in zip(cs, width)) + " |"  # noqa: E731
        return "\n".join([line(head), "|" + "|".join("-" * (w + 2) for w in width) + "|"] +
                         [line(b) for b in body]) + "\n"
    return "\n".join(",".join(r) for r in [head] + body) + "\n"


def random_verify_configs(count: int, seed: int) -> List[LayerConfig]:
    """bench.hpp:164-183: n <= 32, k <= 11, S <= 4, f and f' <= 8."""
    out = []
    for i in range(count):
        def draw(salt, lo, hi):
            h = splitmix64(seed ^ splitmix64((i * 6364136223846793005 + salt) & 0xFFFFFFFFFFFFFFFF))
            return lo + h % (hi - lo + 1)

        image = draw(1, 2, 32)
        kernel = draw(2, 1, min(11, image))
        out.append(LayerConfig(kernel, image, draw(3, 1, 8), draw(4, 1, 8), draw(5, 1, 4)))
    return out


@dataclass
class VerifyResult:  # bench.hpp:152-160
    configs: int = 0
    max_err_forward: float = 0.0
    max_err_grad_input: float = 0.0
    max_err_grad_weight: float = 0.0

    def within(self, tol_fwd: float, tol_gi: float, tol_gw: float) -> bool:
        return (self.max_err_forward <= tol_fwd and self.max_err_grad_input <= tol_gi
                and self.max_err_grad_weight <= tol_gw)


def max_rel_error(got, ref) -> float:
    """tensor.hpp:177-181: max |got - ref| / max(max |ref|, 1e-30)."""
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(got - ref)) / max(float(np.max(np.abs(ref))), 1e-30))


def verify_sweep(cfgs: Sequence[LayerConfig], seed: int,
                 reference: Callable[[str, np.ndarray, np.ndarray], np.ndarray],
                 device: int = 0) -> VerifyResult:
    """bench.hpp:187-222 with the B200 operators as the method under test.
    reference(op, a, b) -> the comparison result for op in
    {"forward", "grad_input", "grad_weight"} (e.g. the direct oracle)."""
    out = VerifyResult(configs=len(cfgs))
    if not cfgs:
        return out
    ws = ConvWorkspace(list(cfgs), device=device)  # one workspace, all configs (:193)
    for cfg in cfgs:
        x, w, gy = make_inputs(cfg, seed)
        out.max_err_forward = max(out.max_err_forward,
                                  max_rel_error(ws.forward(x, w), reference("forward", x, w)))
        out.max_err_grad_input = max(out.max_err_grad_input,
                                     max_rel_error(ws.grad_input(gy, w), reference("grad_input", gy, w)))
        out.max_err_grad_weight = max(out.max_err_grad_weight,
                                      max_rel_error(ws.grad_weight(gy, x), reference("grad_weight", gy, x)))
    return out
