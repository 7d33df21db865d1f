"""Per-stage device times (CUDA events between the 4 launches of each op),
averaged over reps with an L2 flush before each op.  Development tool."""
import argparse
import json
import os
import statistics
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
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--S", type=int, default=0, help="override the batch")
    a = ap.parse_args()
    (k, n, f, fo, S), label = bench.parse_config(a.config)
    S = a.S or S
    no = n - k + 1
    dev = torch.device("cuda:0")
    x = torch.from_numpy(fill_uniform((S, f, n, n), 1234, 1)).to(dev)
    w = torch.from_numpy(fill_uniform((fo, f, k, k), 1234, 2)).to(dev)
    gy = torch.from_numpy(fill_uniform((S, fo, no, no), 1234, 3)).to(dev)
    ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    ops = {"forward": lambda: ws.forward(x, w), "grad_input": lambda: ws.grad_input(gy, w),
           "grad_weight": lambda: ws.grad_weight(gy, x)}
    for fn in ops.values():
        fn()
    ws.set_stage_timing(True)
    out = {}
    for name, fn in ops.items():
        st = []
        for _ in range(a.reps):
            flush.fill_(1.0)
            fn()
            st.append(ws.stage_ms())
        out[name] = [round(statistics.median(v[i] for v in st) * 1000, 2) for i in range(4)]
    out["total_us"] = round(sum(sum(v) for v in out.values()), 1)
    print(json.dumps({"config": a.config, "S": S, "dbg": os.environ.get("FFTCONV_B200_GEMM_DEBUG", "0"),
                      "stage_us[r2cA,r2cB,gemm,c2r]": out}))


if __name__ == "__main__":
    main()
