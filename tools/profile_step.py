"""Minimal driver for ncu: `reps` x (fprop, bprop, accGrad) of one layer on
cuda:0 through the product path, nothing else on the GPU.  Never used for
reported numbers (a number printed under a profiler is not a measurement)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402
from paper_1312_5851_b200.rng import fill_uniform  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--ops", default="forward,grad_input,grad_weight")
    a = ap.parse_args()
    (k, n, f, fo, S), _ = bench.parse_config(a.config)
    no = n - k + 1
    dev = torch.device("cuda:0")
    x = torch.from_numpy(fill_uniform((S, f, n, n), 1234, 1)).to(dev)
    w = torch.from_numpy(fill_uniform((fo, f, k, k), 1234, 2)).to(dev)
    gy = torch.from_numpy(fill_uniform((S, fo, no, no), 1234, 3)).to(dev)
    ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
    ops = a.ops.split(",")
    for _ in range(a.reps):
        if "forward" in ops:
            ws.forward(x, w)
        if "grad_input" in ops:
            ws.grad_input(gy, w)
        if "grad_weight" in ops:
            ws.grad_weight(gy, x)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
