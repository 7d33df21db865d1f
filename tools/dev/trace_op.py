"""Runs one operator of a config once (after a warm-up) with a trace build
(FFTCONV_B200_LIB=lib_alt/libfftconv_trace.so, -DFCB_XFORM_TRACE) so CTA 0's
per-group clock64 timeline is printed.  python tools/dev/trace_op.py paper grad_weight"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402
from paper_1312_5851_b200.rng import fill_uniform  # noqa: E402

cfg, op = sys.argv[1], sys.argv[2]
(k, n, f, fo, S), _ = bench.parse_config(cfg)
S = int(os.environ.get("TRACE_S", S))
no = n - k + 1
dev = torch.device("cuda:0")
x = torch.from_numpy(fill_uniform((S, f, n, n), 1234, 1)).to(dev)
w = torch.from_numpy(fill_uniform((fo, f, k, k), 1234, 2)).to(dev)
gy = torch.from_numpy(fill_uniform((S, fo, no, no), 1234, 3)).to(dev)
ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
ops = {"forward": lambda: ws.forward(x, w), "grad_input": lambda: ws.grad_input(gy, w),
       "grad_weight": lambda: ws.grad_weight(gy, x)}
for i in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    ops[op]()
    torch.cuda.synchronize()
    print("---- call", i, flush=True)
