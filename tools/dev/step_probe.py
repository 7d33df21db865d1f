"""Where does a P step's time go?  Eager step (events), the same three ops
captured in one CUDA graph and replayed, host time per op call, and each op
alone.  Development tool: python tools/dev/step_probe.py [--config paper]"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402
from paper_1312_5851_b200.rng import fill_uniform  # noqa: E402


def ev_time(fn, reps, flush=None):
    out = []
    for i in range(reps):
        if flush is not None:
            flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        out.append((a, b))
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in out)
    return statistics.median(t), t[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--S", type=int, default=0, help="override the batch (a strong-scaling shard)")
    a = ap.parse_args()
    (k, n, f, fo, S), _ = bench.parse_config(a.config)
    S = a.S or S
    no = n - k + 1
    dev = torch.device("cuda:0")
    x = torch.from_numpy(fill_uniform((S, f, n, n), 1234, 1)).to(dev)
    w = torch.from_numpy(fill_uniform((fo, f, k, k), 1234, 2)).to(dev)
    gy = torch.from_numpy(fill_uniform((S, fo, no, no), 1234, 3)).to(dev)
    ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    y = torch.empty((S, fo, no, no), device=dev)
    ops = {"forward": lambda: ws.forward(x, w), "grad_input": lambda: ws.grad_input(gy, w),
           "grad_weight": lambda: ws.grad_weight(gy, x)}

    def step():
        for fn in ops.values():
            fn()

    for _ in range(10):
        step()
    torch.cuda.synchronize()
    print("eager step flushed   median/min us: %.1f / %.1f" % ev_time(step, a.reps, flush))
    print("eager step unflushed median/min us: %.1f / %.1f" % ev_time(step, a.reps))
    for name, fn in ops.items():
        print(f"  {name:12s} flushed %.1f / %.1f   unflushed %.1f / %.1f" % (ev_time(fn, a.reps, flush) +
                                                                            ev_time(fn, a.reps)))
    # host cost per op call (GPU kept busy behind a sleep so the host never waits)
    torch.cuda._sleep(200_000_000)
    host = {}
    for name, fn in ops.items():
        t0 = time.perf_counter()
        for _ in range(20):
            fn()
        host[name] = (time.perf_counter() - t0) / 20 * 1e6
    torch.cuda.synchronize()
    print("host us per call:", {k_: round(v, 1) for k_, v in host.items()})
    # graph capture of one step
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            step()
        torch.cuda.synchronize()
        print("graph step flushed   median/min us: %.1f / %.1f" % ev_time(g.replay, a.reps, flush))
        print("graph step unflushed median/min us: %.1f / %.1f" % ev_time(g.replay, a.reps))
    except Exception as e:
        print("graph capture failed:", e)


if __name__ == "__main__":
    main()
