"""Runs the three operators of one layer `--reps` times (no timing) so ncu
can capture their kernels.  Development tool:

  ncu --set full --clock-control none --import-source on -k regex:'r2c|cgemm|c2r' \
      -s <skip> -c <count> -o gpurun_out/prof python tools/profile_step.py --config paper
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402
from paper_1312_5851_b200.rng import fill_uniform  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="paper")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--ops", default="forward,grad_input,grad_weight")
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
    ops = {"forward": lambda: ws.forward(x, w), "grad_input": lambda: ws.grad_input(gy, w),
           "grad_weight": lambda: ws.grad_weight(gy, x)}
    sel = a.ops.split(",")
    for _ in range(a.reps):
        for name in sel:
            ops[name]()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
