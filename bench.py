#!/usr/bin/env python
"""Benchmark of the FFT convolution layer hot path (BASELINE.json metric).

One step = fprop + bprop + accGrad of one conv layer (the reference's three
ConvWorkspace operators, conv_fft.hpp:74-206) over the layer's full
minibatch, every transform recomputed from spatial data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config paper|wide|small|sweep:n,k]
                  [--impl ours|reference]

N>1 runs one process per GPU under torchrun: the minibatch S is sharded
(strong scaling: the layer's S stays fixed), fprop/bprop are local and
accGrad's weight gradient is summed with an NCCL all-reduce.  Rank 0 prints
one JSON line.  Timing: CUDA events on the launching stream, L2 flushed
between steps (256 MiB write), max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

CONFIGS = {
    # BASELINE.json configs (k, n, f, f', S)
    "small": (5, 32, 16, 16, 8),
    "paper": (7, 32, 96, 96, 128),
    "wide": (11, 64, 256, 256, 128),
    # configs[4]'s first layer (f = 3 -> 96, n = 128; FFT size 128)
    "alex1": (11, 128, 3, 96, 128),
}
METRIC = "ms per fprop+bprop+accGrad per layer (S=128) + direct-conv-equiv TFLOP/s"
OPS = ("forward", "grad_input", "grad_weight")


def parse_config(name):
    if name.startswith("sweep:"):
        n, k = (int(v) for v in name.split(":")[1].split(","))
        return (k, n, 96, 96, 128), f"kernel/input sweep point S=128 f=f'=96 n={n} k={k}"
    k, n, f, fo, S = CONFIGS[name]
    label = {"paper": "paper sweep point", "wide": "wide layer", "small": "small layer",
             "alex1": "AlexNet-style first layer"}[name]
    return CONFIGS[name], f"{label} S={S} f={f} f'={fo} n={n} k={k}"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled in the background.

    Two sampler processes: the SM clock every 50 ms, the throttle reasons
    every 250 ms.  The reasons and utilization queries stall the host driver
    calls briefly (measured: with them at 50 ms, host-driven layer-stack
    iterations took 10-150 ms outliers in the timed region; clocks alone
    never did, tools/dev/smi_probe.sh, tools/dev/stack_rep.sh), so the
    reasons run 5x less often and utilization is not sampled (the samplers
    run only around the timed steps, so every sample is under load)."""

    QF = "timestamp,clocks.sm,clocks.max.sm"
    QR = ("timestamp,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
          "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index, reasons_during=True, during=True):
        self.index = index
        self.reasons_during = reasons_during  # False: one reasons query right after the steps
        self.during = during  # False: no background sampling, one query before and one after
        self.snaps = []
        self.procs = []
        self.paths = []
        self.t0 = self.t1 = None  # the loaded window (begin() / end()); samples outside it are dropped

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def _in_window(self, rows):
        if self.t0 is None or self.t1 is None:
            return rows
        import datetime

        keep = []
        for r in rows:
            try:
                ts = datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            if self.t0 <= ts <= self.t1:
                keep.append(r)
        return keep or rows

    def _spawn(self, q, lms):
        fd, path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
             "-lms", str(lms), "-f", path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        self.procs.append(proc)
        self.paths.append(path)

    def _snap(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QF},{self.QR}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=10).stdout
            for line in out.splitlines():
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    self.snaps.append(parts)
        except Exception:
            pass

    def start(self):
        if os.environ.get("FFTCONV_BENCH_NO_SMI") == "1":  # diagnostics: no sampler process
            return
        if not self.during:
            self._snap()
            return
        try:
            self._spawn(self.QF, 50)
            if self.reasons_during:
                self._spawn(self.QR, 250)
            # nvidia-smi's start-up (NVML init) stalls the driver for a moment:
            # let both finish it before the timed region
            t_end = time.time() + 3.0
            while time.time() < t_end and any(os.path.getsize(p) == 0 and pr.poll() is None
                                               for p, pr in zip(self.paths, self.procs)):
                time.sleep(0.02)
            time.sleep(0.1)
        except Exception:
            self.procs, self.paths = [], []

    @staticmethod
    def _rows(path, width):
        rows = []
        try:
            with open(path) as fh:
                for line in fh:
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) >= width:
                        rows.append(parts)
            os.unlink(path)
        except OSError:
            pass
        return rows

    def stop(self):
        if not self.during:
            self._snap()
            if not self.snaps:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            sm = [float(r[1]) for r in self.snaps if r[1].replace(".", "").isdigit()]
            return {"sm_mhz": statistics.median(sm) if sm else None,
                    "sm_max_mhz": float(self.snaps[0][2]) if self.snaps[0][2].replace(".", "").isdigit() else None,
                    "reasons": sorted({names[i] for r in self.snaps for i in range(4) if r[4 + i] == "Active"}),
                    "samples": len(self.snaps),
                    "note": "one query right before and one right after the timed steps (background "
                            "nvidia-smi sampling stalls these host-driven steps)"}
        if len(self.procs) != (2 if self.reasons_during else 1):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if not self.reasons_during:  # the GPU is still warm: one query of the current reasons
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QR}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
                once = [[p.strip() for p in line.split(",")] for line in out.splitlines() if line.strip()]
            except Exception:
                once = []
        for proc in self.procs:
            proc.terminate()
            try:
                proc.wait(timeout=5)
            except Exception:
                proc.kill()
        rows = self._rows(self.paths[0], 3)
        rrows = self._in_window(self._rows(self.paths[1], 5)) if self.reasons_during else \
            [r for r in once if len(r) >= 5]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = self._in_window(rows)  # samples inside the loaded window only
        sm = [float(r[1]) for r in loaded if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rrows for i in range(4) if r[1 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(loaded),
                "reason_samples": len(rrows)}


# ---------------------------------------------------------------- reference arm
def cpu_reference_step_ms(cfg, iters, warmup, threads, seed=1234):
    """Reference run_op_bench<float> (bench.hpp:80-145), FFT method, per op."""
    import oracle

    k, n, f, fo, S = cfg
    out = {}
    for op_i, op in enumerate(OPS):
        r = oracle.ref_run_op_bench(k, n, f, fo, S, op_i, 1, iters, warmup, threads, seed)
        out[op] = r["mean_ms"]
    return out


def cpu_model():
    """The host CPU's model name (lscpu's, from /proc/cpuinfo)."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_threads():
    import oracle

    return int(oracle.ref_lib().ref_resolve_threads(0))


def run_reference_arm(args, cfg, label):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfftconv_ref.so not built"}))
        return
    threads = cpu_threads()
    k, n, f, fo, S = cfg
    # Each step: the reference's own run_op_bench per operator (workspace and
    # inputs built outside its clock, bench.hpp:100-142), one warm-up + one
    # timed call; the step time is the sum of the three timed operators.
    for _ in range(args.warmup):
        cpu_reference_step_ms(cfg, 1, 0, threads)
    steps = []
    for _ in range(args.steps):
        steps.append(sum(cpu_reference_step_ms(cfg, 1, 1, threads).values()))
    ms = statistics.mean(steps)
    E = 2 * S * f * fo * (n - k + 1) ** 2 * k * k
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference fill_uniform, seed 1234)",
        "config": {"workload": label, "k": k, "n": n, "f": f, "f_prime": fo, "S": S},
        "run": {"parallelism": f"reference CPU (std::thread parallel_for, {threads} threads)"},
        "impl": "reference",
        "tflops_equiv": 3 * E / (ms * 1e-3) / 1e12,
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                         "sample": f"reference run_op_bench<float> (FFT method) fprop+bprop+accGrad on the "
                                   f"full layer, {args.steps} steps (1 warm-up + 1 timed call per operator "
                                   f"each) after {args.warmup} warm-up steps"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def main():
    if os.environ.get("FFTCONV_B200_WATCHDOG"):  # debugging aid: dump stacks if stuck
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["FFTCONV_B200_WATCHDOG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="paper")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--strong", action="store_true",
                    help="N>1: split the S-sample minibatch across ranks (the default; kept for compatibility)")
    ap.add_argument("--weak", action="store_true",
                    help="N>1: weak scaling instead -- every rank holds a full S-sample shard of an N*S minibatch")
    ap.add_argument("--chunks", type=int, default=4,
                    help="N>1: f'-chunks of accGrad's c2r, each all-reduced while the next transforms")
    ap.add_argument("--dist-backend", default="nccl",
                    help="nccl (one GPU per rank); gloo lets ranks share a GPU for testing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config.startswith("stack"):
        return run_stack(args)
    cfg, label = parse_config(args.config)
    if args.impl == "reference":
        return run_reference_arm(args, cfg, label)

    import torch
    import torch.distributed as dist

    from paper_1312_5851_b200 import ConvWorkspace, LayerConfig
    from paper_1312_5851_b200.rng import ROLE_GRAD_OUTPUT, ROLE_INPUT, ROLE_WEIGHTS, fill_uniform
    from paper_1312_5851_b200.sharded import shard_range
    from paper_1312_5851_b200 import cost_model
    from paper_1312_5851_b200._native import gemm_kind

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.dist_backend == "nccl":
            # NCCL init lines in the log (nranks / NVLink / NVLS) for the driver
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)

    k, n, f, fo, S = cfg
    no = n - k + 1
    # Strong scaling (default, BASELINE configs[3] / the north star: "the
    # minibatch S is sharded across the GPUs"): the S-sample minibatch is
    # split across the ranks.  --weak: every rank holds a full S-sample shard
    # of an N*S-sample minibatch (per-GPU work fixed).
    weak = args.weak and world > 1
    S_glob = S * world if weak else S
    b0, b1 = shard_range(S_glob, world, rank)
    Sl = b1 - b0
    lcfg = LayerConfig(k, n, f, fo, Sl)
    # Inputs: the reference generator (same bytes the CPU path consumes), this
    # rank's minibatch slice, resident in HBM before timing starts.
    x = fill_uniform((Sl, f, n, n), 1234, ROLE_INPUT, offset=b0 * f * n * n)
    w = fill_uniform((fo, f, k, k), 1234, ROLE_WEIGHTS)
    gy = fill_uniform((Sl, fo, no, no), 1234, ROLE_GRAD_OUTPUT, offset=b0 * fo * no * no)
    xd, wd, gyd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, w, gy))
    ws = ConvWorkspace([lcfg], device=local)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    sc = None
    if world > 1:
        from paper_1312_5851_b200.sharded import NcclComm, ShardedConv

        # accGrad's gw all-reduce through the library (NCCL, chunked behind
        # the c2r); gloo (ranks sharing a GPU in tests) reduces via torch
        comm = NcclComm(local) if args.dist_backend == "nccl" else None
        sc = ShardedConv(ws, comm=comm, chunks=args.chunks)

    def step(reduce=True):
        if sc is not None and reduce:
            return sc.forward(xd, wd), sc.grad_input(gyd, wd), sc.grad_weight(gyd, xd)
        return ws.forward(xd, wd), ws.grad_input(gyd, wd), ws.grad_weight(gyd, xd)

    # warm-up (also brings clocks up)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # time-based loops run a rank-dependent number of steps: no collectives there
    t_end = time.time() + 1.0
    while time.time() < t_end:
        step(reduce=False)
        flush.fill_(1.0)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    # keep the GPU busy while the sampler spins up, then the timed steps
    t_end = time.time() + 0.5
    sampler.begin()
    while time.time() < t_end:
        step(reduce=False)
        flush.fill_(1.0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        flush.fill_(float(len(times)))  # evict L2 between timed steps (untimed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        times.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in times]
    # hold load a little longer so the sampler sees the clocks under load
    t_end = time.time() + 0.3
    while time.time() < t_end:
        step(reduce=False)
        flush.fill_(1.0)
    torch.cuda.synchronize()
    sampler.end()
    clocks = sampler.stop()
    ms = statistics.mean(step_ms)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    launches_per_step = 0
    for fn in (lambda: ws.forward(xd, wd), lambda: ws.grad_input(gyd, wd), lambda: ws.grad_weight(gyd, xd)):
        fn()
        launches_per_step += ws.last_launch_count()
    torch.cuda.synchronize()

    # ---- per-kernel device times (events between the launches of each op)
    ws.set_stage_timing(True)
    stage = {op: [] for op in OPS}
    gemm_path = {}  # the GEMM kernel that actually ran per op (auto may pick either)
    for _ in range(5):
        for op, fn in (("forward", lambda: ws.forward(xd, wd)), ("grad_input", lambda: ws.grad_input(gyd, wd)),
                       ("grad_weight", lambda: ws.grad_weight(gyd, xd))):
            flush.fill_(2.0)
            fn()
            stage[op].append(ws.stage_ms())
            gemm_path[op] = ws.last_gemm_path() or "tf32x3"
    # ---- live per-kernel spans with the PDL chain intact (in-kernel global
    # timer: first CTA past its dependency wait -> last CTA done), the same
    # flushed single-operator calls as the event stage timings above
    live = None
    try:
        ws.set_span_timing(True)
        for _ in range(5):
            for op, fn in (("forward", lambda: ws.forward(xd, wd)), ("grad_input", lambda: ws.grad_input(gyd, wd)),
                           ("grad_weight", lambda: ws.grad_weight(gyd, xd))):
                flush.fill_(3.0)
                fn()
        spans = ws.span_ms(15)
        ws.set_span_timing(False)
        live = {op: [statistics.mean(sp[i][k] for i in range(j, len(spans), 3)) if all(
            sp[i][k] is not None for i in range(j, len(spans), 3)) else None for k in range(3)]
            for j, op in enumerate(OPS) for sp in [spans]}
    except Exception as exc:  # reported, never fatal
        live = {"error": str(exc)}
    comm_stats = None
    if sc is not None:
        # the sharded accGrad: collective span, the part not hidden behind the
        # chunked c2r, and the whole sharded op (all ranks run the same count)
        spans, exposed, op_ms = [], [], []
        for _ in range(5):
            flush.fill_(2.0)
            dist.barrier()
            torch.cuda.synchronize()
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            sc.grad_weight(gyd, xd)
            b_.record(stream)
            torch.cuda.synchronize()
            op_ms.append(a_.elapsed_time(b_))
            if sc.comm is not None:
                sp, ex = sc.comm_ms()
                spans.append(sp)
                exposed.append(ex)
        t = torch.tensor([statistics.mean(op_ms), statistics.mean(spans) if spans else 0.0,
                          statistics.mean(exposed) if exposed else 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sharded_ms, ar_ms, ar_exposed = (float(v) for v in t.tolist())
        comm_stats = {"grad_weight_sharded_ms": sharded_ms, "allreduce_ms": ar_ms if sc.comm else None,
                      "allreduce_exposed_ms": ar_exposed if sc.comm else None,
                      "allreduce_hidden_frac": (1.0 - ar_exposed / ar_ms) if (sc.comm and ar_ms > 0) else None,
                      "allreduce_bytes": 4 * fo * f * k * k, "chunks": args.chunks,
                      "path": ("fftconv_b200_grad_weight_sharded: c2r in f'-chunks, each chunk's gw rows "
                               "ncclAllReduce'd on a side stream (library-owned communicator)")
                      if sc.comm else "torch.distributed all_reduce of gw (gloo)",
                      "max_over_ranks": True}
    ws.set_stage_timing(False)
    stage_ms = {op: [statistics.mean(v[i] for v in stage[op]) for i in range(4)] for op in OPS}

    hbm_gbs, bf16_tflops, peak_src = load_peaks()
    kind = gemm_kind()
    op_tflops = {op: cost_model.gemm_tensor_tflops(bf16_tflops, gemm_path[op]) for op in OPS}
    lc = lcfg
    bins = lc.bins()
    # algorithmic bytes per launch of each transform kernel, flops of the GEMM
    Sl_, f_, fo_ = Sl, f, fo
    alg = {
        "forward": [4 * Sl_ * f_ * n * n + 8 * bins * Sl_ * f_, 4 * fo_ * f_ * k * k + 8 * bins * fo_ * f_,
                    8 * bins * Sl_ * f_ * fo_, 8 * bins * Sl_ * fo_ + 4 * Sl_ * fo_ * no * no],
        "grad_input": [4 * Sl_ * fo_ * no * no + 8 * bins * Sl_ * fo_, 4 * fo_ * f_ * k * k + 8 * bins * fo_ * f_,
                       8 * bins * Sl_ * f_ * fo_, 8 * bins * Sl_ * f_ + 4 * Sl_ * f_ * n * n],
        "grad_weight": [4 * Sl_ * fo_ * no * no + 8 * bins * Sl_ * fo_, 4 * Sl_ * f_ * n * n + 8 * bins * Sl_ * f_,
                        8 * bins * Sl_ * f_ * fo_, 8 * bins * f_ * fo_ + 4 * fo_ * f_ * k * k],
    }
    kname = ["r2c(A)", "r2c(B)", "cgemm_bins_tcgen05", "c2r"]
    stages = []
    for op in OPS:
        merged = stage_ms[op][1] < 0.005  # both forward transforms in one launch
        for i in range(4):
            t_ms = stage_ms[op][i]
            if merged and i == 1:
                continue
            if merged and i == 0:
                ach = (alg[op][0] + alg[op][1]) / (t_ms * 1e-3) / 1e9
                stages.append({"op": op, "kernel": "r2c(A+B)", "ms": t_ms, "bound": "hbm", "achieved": ach,
                               "peak": hbm_gbs, "unit": "GB/s", "frac": ach / hbm_gbs,
                               "alg_bytes": alg[op][0] + alg[op][1]})
                continue
            if i == 2:  # bound by whichever floor is larger: tensor passes or operand/product bytes
                gb = cost_model.gemm_bytes(lc)
                gemm_tflops = op_tflops[op]
                if alg[op][i] / (gemm_tflops * 1e12) >= gb / (hbm_gbs * 1e9):
                    ach = alg[op][i] / (t_ms * 1e-3) / 1e12
                    stages.append({"op": op, "kernel": kname[i], "ms": t_ms, "bound": "tensor", "achieved": ach,
                                   "peak": gemm_tflops, "unit": "TFLOP/s", "frac": ach / gemm_tflops,
                                   "alg_flops": alg[op][i], "gemm_kind": gemm_path[op]})
                else:
                    ach = gb / (t_ms * 1e-3) / 1e9
                    stages.append({"op": op, "kernel": kname[i], "ms": t_ms, "bound": "hbm", "achieved": ach,
                                   "peak": hbm_gbs, "unit": "GB/s", "frac": ach / hbm_gbs, "alg_bytes": gb,
                                   "alg_flops": alg[op][i], "gemm_kind": gemm_path[op]})
            else:
                ach = alg[op][i] / (t_ms * 1e-3) / 1e9
                stages.append({"op": op, "kernel": kname[i], "ms": t_ms, "bound": "hbm", "achieved": ach,
                               "peak": hbm_gbs, "unit": "GB/s", "frac": ach / hbm_gbs, "alg_bytes": alg[op][i]})
    # the same fractions from the live spans (PDL chain intact)
    stages_live, roofline_live = None, None
    if live and "error" not in live and all(v is not None for op in OPS for v in live[op]):
        stages_live = []
        for op in OPS:
            k1, k3, k4 = live[op]
            b1 = alg[op][0] + alg[op][1]
            gb = cost_model.gemm_bytes(lc)
            t_floor_gemm = max(alg[op][2] / (op_tflops[op] * 1e12), gb / (hbm_gbs * 1e9))
            stages_live.append({"op": op, "kernel": "r2c(A+B)", "ms": k1, "achieved": b1 / (k1 * 1e-3) / 1e9,
                                "unit": "GB/s", "frac": b1 / (k1 * 1e-3) / 1e9 / hbm_gbs})
            stages_live.append({"op": op, "kernel": "cgemm_bins_tcgen05", "ms": k3,
                                "frac": t_floor_gemm / (k3 * 1e-3)})
            stages_live.append({"op": op, "kernel": "c2r", "ms": k4, "achieved": alg[op][3] / (k4 * 1e-3) / 1e9,
                                "unit": "GB/s", "frac": alg[op][3] / (k4 * 1e-3) / 1e9 / hbm_gbs})
        r2c_live = [st_ for st_ in stages_live if st_["kernel"] == "r2c(A+B)"]
        ms_r2c = statistics.mean(st_["ms"] for st_ in r2c_live)
        b_r2c = statistics.mean(alg[op][0] + alg[op][1] for op in OPS)
        roofline_live = {"kernel": "r2c_tma_kernel", "bound": "hbm", "achieved": b_r2c / (ms_r2c * 1e-3) / 1e9,
                         "peak": hbm_gbs, "unit": "GB/s", "frac": b_r2c / (ms_r2c * 1e-3) / 1e9 / hbm_gbs,
                         "transform_frac_per_pass": {
                             op: (sum(alg[op][i] for i in (0, 1, 3)) / ((live[op][0] + live[op][2]) * 1e-3) / 1e9)
                             / hbm_gbs for op in OPS},
                         "note": "per-kernel spans from the kernels' own global-timer stamps with the "
                                 "programmatic-dependent-launch chain intact (the event stage timings above "
                                 "break it, so each of those includes a full launch gap)"}
    # dominant kernel = largest total time across the step (the m = 128
    # transforms are two kernels each, fft_large.cuh)
    m_fft = 1 << max(0, (n - 1).bit_length())
    xf_names = ({"r2c": "r2c128_cols_kernel+r2c128_rows_kernel", "c2r": "c2r128_rows_kernel+c2r128_cols_kernel"}
                if m_fft == 128 else {"r2c": "r2c_tma_kernel", "c2r": "c2r_tma_kernel"})
    tot = {}
    for s_ in stages:
        key = xf_names.get(s_["kernel"][:3], s_["kernel"])
        tot[key] = tot.get(key, 0.0) + s_["ms"]
    dom = max(tot, key=tot.get)
    dom_st = [s_ for s_ in stages if xf_names.get(s_["kernel"][:3], s_["kernel"]) == dom]
    dom_ms = statistics.mean(s_["ms"] for s_ in dom_st)
    if dom == "cgemm_bins_tcgen05" and dom_st[0]["bound"] == "tensor":
        alg_per_launch = statistics.mean(s_["alg_flops"] for s_ in dom_st)
        achieved = alg_per_launch / (dom_ms * 1e-3) / 1e12
        peak_t = statistics.mean(s_["peak"] for s_ in dom_st)
        kinds = sorted({s_["gemm_kind"] for s_ in dom_st})
        basis = " / ".join("/ 3 (fp16x3 passes)" if k_ == "f16x3" else "/ 2 (TF32 rate) / 3 (3xTF32 passes)"
                           for k_ in kinds)
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s",
                    "frac": achieved / peak_t,
                    "peak_basis": f"{peak_src} bf16 {bf16_tflops} TF/s {basis}"}
    else:
        alg_per_launch = statistics.mean(s_["alg_bytes"] for s_ in dom_st)
        achieved = alg_per_launch / (dom_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                    "frac": achieved / hbm_gbs, "peak_basis": peak_src}
    roofline["kernel"] = dom
    roofline["share_of_step"] = tot[dom] / sum(tot.values())
    roofline["traffic"] = ncu_traffic(dom, args.config)

    # ---- end to end through the public API with host (pinned) buffers
    e2e = None
    if world == 1:
        def pinned(shape):
            return torch.empty(shape, dtype=torch.float32).pin_memory().numpy()

        xp, wp, gyp = pinned(x.shape), pinned(w.shape), pinned(gy.shape)
        xp[...], wp[...], gyp[...] = x, w, gy
        y_h, gx_h, gw_h = pinned((Sl, fo, no, no)), pinned((Sl, f, n, n)), pinned((fo, f, k, k))
        for _ in range(2):
            ws.forward(xp, wp, out=y_h), ws.grad_input(gyp, wp, out=gx_h), ws.grad_weight(gyp, xp, out=gw_h)
        e2e_ms = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            ws.forward(xp, wp, out=y_h)
            ws.grad_input(gyp, wp, out=gx_h)
            ws.grad_weight(gyp, xp, out=gw_h)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = 4 * (x.size + w.size + gy.size + w.size + gy.size + x.size)
        d2h = 4 * (y_h.size + gx_h.size + gw_h.size)
        # the PCIe floor of this traffic on this box: pinned copies of the same
        # sizes, each direction alone (the step's three calls are synchronous)
        def copy_ms(nbytes, to_dev):
            hbuf = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
            dbuf = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
            best = 1e9
            for _ in range(3):
                t0 = time.perf_counter()
                (dbuf.copy_(hbuf, non_blocking=True) if to_dev else hbuf.copy_(dbuf, non_blocking=True))
                torch.cuda.synchronize()
                best = min(best, (time.perf_counter() - t0) * 1e3)
            return best
        h2d_ms, d2h_ms = copy_ms(int(h2d), True), copy_ms(int(d2h), False)
        e2e = {"value": statistics.mean(e2e_ms), "unit": "ms", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "pcie_floor_ms": {"h2d_alone": h2d_ms, "d2h_alone": d2h_ms,
                                 "h2d_GBps": h2d / h2d_ms / 1e6, "d2h_GBps": d2h / d2h_ms / 1e6},
               "path": "ConvWorkspace.forward/grad_input/grad_weight(out=) on pinned numpy -> "
                       "fftconv_b200_*_host C ABI; each call pipelined over minibatch chunks "
                       "(H2D / compute / D2H on three streams), synchronous per call"}

    # ---- CPU reference beside it (rank 0, N=1 only), and the reference's
    # own bench protocol (bench.hpp:80-145) for both implementations
    cpu = None
    protocol = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            from paper_1312_5851_b200 import harness

            if oracle.ref_available():
                threads = cpu_threads()
                iters = 1 if args.config == "wide" else 2
                lcfg_full = LayerConfig(k, n, f, fo, S)
                ref_rows = []
                per_op = {}
                for op_i, op in enumerate(OPS):
                    st = oracle.ref_run_op_bench(k, n, f, fo, S, op_i, 1, iters, 1, threads, 1234)
                    per_op[op] = st["mean_ms"]
                    ref_rows.append(("fft", op_i, iters, st))
                cpu = {"value": sum(per_op.values()), "unit": "ms", "cores": threads, "kind": "reference",
                       "cpu_model": cpu_model(), "per_op_ms": per_op,
                       "sample": f"reference run_op_bench<float> (FFT method) on the full layer, {iters} iters "
                                 f"after 1 warm-up per op"}
                if args.config in ("small", "paper"):
                    # Method::direct beside it; one timed call per op (P: ~3 x 5 s)
                    dper = {}
                    for op_i, op in enumerate(OPS):
                        st = oracle.ref_run_op_bench(k, n, f, fo, S, op_i, 0, 1, 0, threads, 1234)
                        dper[op] = st["mean_ms"]
                        ref_rows.append(("direct", op_i, 1, st))
                    cpu["direct"] = {"value": sum(dper.values()), "unit": "ms", "per_op_ms": dper,
                                     "sample": "reference run_op_bench<float> (direct method), 1 timed call per op"}
                # our operators under the same protocol (device-resident, CUDA events per call)
                ours = [harness.run_op_bench(lcfg_full, harness.BenchOp(i), iters=10, warmup=3, seed=1234,
                                             resident=True, device=local) for i in range(3)]
                rows = list(ours)
                for method, op_i, it, st in ref_rows:
                    r_ = harness.BenchResult(harness.BenchOp(op_i), method, lcfg_full, it, 1 if method == "fft" else 0,
                                             threads, 1234, harness.BenchStats(st["mean_ms"], st["std_ms"],
                                                                               st["min_ms"], st["median_ms"]),
                                             st["checksum"])
                    rows.append(r_)
                ref_ck = {r_.op: r_.checksum for r_ in rows if r_.method == "fft"}
                protocol = {
                    "b200": {OPS[int(r_.op)]: {"mean_ms": r_.stats.mean_ms, "std_ms": r_.stats.std_ms,
                                               "min_ms": r_.stats.min_ms, "median_ms": r_.stats.median_ms,
                                               "checksum": r_.checksum,
                                               "checksum_rel_diff_vs_reference":
                                                   abs(r_.checksum - ref_ck[r_.op]) / max(abs(ref_ck[r_.op]), 1e-30)}
                             for r_ in ours},
                    "csv": harness.bench_table(rows, "csv"),
                    "note": "rows in the reference CLI schema (fftconv_cli.cpp:144-149): method b200 = this "
                            "implementation (device-resident, per-call CUDA events), fft / direct = the "
                            "reference's run_op_bench<float> on the host cores",
                }
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "reference", "sample": f"failed: {exc}"}

    # fusion-proof pass-level roofline: sum of the stage
    # floors at the measured peaks over the measured pass time

    stage_us = {op: {"r2c": 1e3 * (stage_ms[op][0] + (0.0 if stage_ms[op][1] < 0.005 else stage_ms[op][1])),
                     "gemm": 1e3 * stage_ms[op][2],
                     "c2r": 1e3 * stage_ms[op][3]} for op in OPS}
    pass_roof = {op: {k: round(v, 4) for k, v in
                      cost_model.roofline_report(lcfg, {op: stage_us[op]}, hbm_gbs, op_tflops[op])[op].items()}
                 for op in OPS}

    E = 2 * S * f * fo * no * no * k * k
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False,
        "scaling": "weak" if weak else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference fill_uniform, seed 1234)",
        # the workload only (identical in both arms); how it ran is in "run"
        "config": {"workload": label, "k": k, "n": n, "f": f, "f_prime": fo, "S": S_glob},
        "run": {"global_batch": S_glob, "S_per_gpu": Sl,
                "parallelism": f"dp{world} (minibatch-sharded, NCCL all-reduce of gw)" if world > 1 else "dp1",
                "l2": "flushed between timed steps (256 MiB write)"},
        "tflops_equiv": 3 * E / (ms * 1e-3) / 1e12,
        "gemm_kind": kind,
        "gemm_path": gemm_path,
        "per_op_ms": {op: sum(stage_ms[op]) for op in OPS},
        "roofline": roofline,
        "pass_roofline": pass_roof,
        "stages": stages,
        "stages_live": stages_live,
        "roofline_live": roofline_live,
        "gpu_launches": launches_per_step * args.steps,
        "multi_gpu": comm_stats,
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "protocol": protocol,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        _teardown(sc.comm if sc is not None else None)


def run_stack(args):
    """--config stack[:preset]: one full training iteration (forward through
    all stages, loss, backward with every weight gradient) of a layer-stack
    preset (layers.hpp:321-348, run_iteration :441-609) on one GPU; the
    reference arm runs the reference's own run_iteration on the host cores."""
    import oracle
    from paper_1312_5851_b200 import layers

    name = args.config.split(":", 1)[1] if ":" in args.config else "reference-net"
    spec = layers.preset_network(name)
    S, seed = spec.default_batch, 1234
    metric = f"ms per training iteration ({name} preset, S={S})"
    base = {"metric": metric, "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference init_params / make_batch, seed 1234)",
            "config": {"workload": f"{name}: " + "; ".join(
                f"conv {s.conv.kernel} {s.conv.image} {s.conv.in_maps} {s.conv.out_maps}" if s.kind == 0
                else ("fc %d" % s.fc_outputs if s.kind == 3 else s.kind.name) for s in spec.stages),
                "S": S, "parallelism": "dp1"}}
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        th = cpu_threads()
        t = []
        for _ in range(max(1, args.steps)):
            _, r = oracle.ref_run_iteration(spec.records(), S, seed, engine=1, threads=th)
            t.append(r["update_output_ms"] + r["update_grad_input_ms"] + r["acc_grad_ms"])
        ms = statistics.mean(t)
        line = dict(base, value=ms, ms_per_step=ms, impl="reference",
                    cpu_baseline={"value": ms, "unit": "ms", "cores": th, "kind": "reference",
                                  "sample": f"reference run_iteration<float> (FFT engine), {len(t)} iterations"},
                    e2e={"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    import torch
    import torch.distributed as dist

    from paper_1312_5851_b200.sharded import NcclComm, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if world > 1:
        # data-parallel step (BASELINE configs[4] on N GPUs): the S-sample
        # minibatch split over the ranks, every gradient summed
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
            comm = NcclComm(local)
        else:
            dist.init_process_group(args.dist_backend)
    b0, b1 = shard_range(S, world, rank)
    params = layers.init_params(spec, seed)
    batch = torch.from_numpy(np.ascontiguousarray(layers.make_batch(spec, S, seed)[b0:b1])).to(dev)
    ws = __import__("paper_1312_5851_b200").ConvWorkspace(spec.conv_configs(b1 - b0), device=local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(args.warmup):
        layers.run_iteration(spec, params, batch, ws=ws, device=local, comm=comm)
    cats = {"update_output_ms": [], "update_grad_input_ms": [], "acc_grad_ms": []}
    wall, launches = [], []
    # the stack's steps are host-driven (hundreds of launches each): any
    # nvidia-smi query during them can stall the host driver calls (10-150 ms
    # outliers, tools/dev/stack_rep.sh), so clocks and reasons are read once
    # right before and once right after the timed steps
    sampler = ClockSampler(local, during=False)
    sampler.start()
    # the categories are CUDA-event spans around host-issued calls: a Python
    # garbage-collection pause inside one (the iteration allocates thousands
    # of objects) idles the GPU and lands in the span, so collect up front
    import gc
    gc.collect()
    gc.disable()
    sampler.begin()
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        r = layers.run_iteration(spec, params, batch, ws=ws, device=local, comm=comm)
        wall.append((time.perf_counter() - t0) * 1e3)
        launches.append(r.gpu_launches)
        for k in cats:
            cats[k].append(getattr(r.times, k))
    sampler.end()
    gc.enable()
    clocks = sampler.stop()
    per = {k: statistics.mean(v) for k, v in cats.items()}
    if world > 1:  # device times, max over ranks
        t = torch.tensor([per[k] for k in cats], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = dict(zip(cats, (float(v) for v in t.tolist())))
        base["n_gpus"] = world
        base["config"]["parallelism"] = (f"dp{world} (minibatch-sharded; conv gw all-reduced by "
                                         f"fftconv_b200_grad_weight_sharded behind the backward pass)")
        base["run"] = {"S_per_gpu": b1 - b0, "global_batch": S}
    ms = sum(per.values())
    if rank != 0:
        if world > 1:
            _teardown(comm)
        return
    line = dict(base, value=ms, ms_per_step=ms, per_category_ms=per,
                wall_ms_incl_param_upload=statistics.mean(wall), loss=r.loss, grad_checksum=r.grad_checksum,
                clocks=clocks, gpu_launches=sum(launches),
                note="value = device time of the three reference categories (CUDA events); conv stages on the "
                     "B200 kernels, relu/pool/fit_to on the layer-stack kernels, fc on fp32 cuBLAS")
    print(json.dumps(line), flush=True)
    if world > 1:
        _teardown(comm)


def _teardown(comm):
    """Every rank destroys the library's NCCL communicator while all ranks are
    still alive, then the process group."""
    import torch
    import torch.distributed as dist

    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
        comm.close()
    dist.destroy_process_group()


def ncu_traffic(kernel, config):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_summary.json), or None when not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(config, {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


if __name__ == "__main__":
    main()
