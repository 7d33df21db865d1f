"""Dev probe: run one operator of a bench config N times and sync (crash hunting).

  python tools/op_probe.py <config> <forward|grad_input|grad_weight> [reps] [S]
"""
import sys

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402

(k, n, f, fo, S), _ = bench.parse_config(sys.argv[1])
op = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if len(sys.argv) > 4:
    S = int(sys.argv[4])
no = n - k + 1
d = torch.device('cuda:0')
x = torch.rand(S, f, n, n, device=d) - 0.5
w = torch.rand(fo, f, k, k, device=d) - 0.5
gy = torch.rand(S, fo, no, no, device=d) - 0.5
ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
fn = {"forward": lambda: ws.forward(x, w), "grad_input": lambda: ws.grad_input(gy, w),
      "grad_weight": lambda: ws.grad_weight(gy, x)}[op]
for _ in range(reps):
    fn()
    torch.cuda.synchronize()
print(op, S, "ok", flush=True)
