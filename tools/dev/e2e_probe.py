"""Dev probe: per-call wall time of the host-pointer operators (pinned
buffers) against the PCIe time of the same bytes."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402

(k, n, f, fo, S), _ = bench.parse_config(sys.argv[1] if len(sys.argv) > 1 else "paper")
no = n - k + 1


def pinned(shape):
    return torch.empty(shape, dtype=torch.float32).pin_memory().numpy()


x, w, gy = pinned((S, f, n, n)), pinned((fo, f, k, k)), pinned((S, fo, no, no))
for a in (x, w, gy):
    a[...] = np.random.default_rng(0).uniform(-1, 1, a.shape)
y, gx, gw = pinned((S, fo, no, no)), pinned((S, f, n, n)), pinned((fo, f, k, k))
ws = ConvWorkspace([LayerConfig(k, n, f, fo, S)], device=0)
ops = {"forward": (lambda: ws.forward(x, w, out=y), x.nbytes + w.nbytes, y.nbytes),
       "grad_input": (lambda: ws.grad_input(gy, w, out=gx), gy.nbytes + w.nbytes, gx.nbytes),
       "grad_weight": (lambda: ws.grad_weight(gy, x, out=gw), gy.nbytes + x.nbytes, gw.nbytes)}
for name, (fn, hin, hout) in ops.items():
    for _ in range(2):
        fn()
    t = []
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        t.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:12s} {statistics.median(t):7.3f} ms   H2D {hin/55e6:6.3f} ms  D2H {hout/56e6:6.3f} ms", flush=True)
