"""Per-operator rel-L2 error vs the reference's ConvWorkspace<double> for one
layer, ours and the reference's own fp32 path: python tools/dev/acc_cfg.py k n f fo S"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402

key = tuple(int(v) for v in sys.argv[1:6])
k, n, f, fo, S = key
no = n - k + 1
x = oracle.fill_uniform((S, f, n, n), 1234, 1)
w = oracle.fill_uniform((fo, f, k, k), 1234, 2)
gy = oracle.fill_uniform((S, fo, no, no), 1234, 3)
th = int(oracle.ref_lib().ref_resolve_threads(0))
r64 = oracle.RefWorkspace([key], dtype=np.float64)
r32 = oracle.RefWorkspace([key], dtype=np.float32)
a = [r64.forward(x, w, th), r64.grad_input(gy, w, th), r64.grad_weight(gy, x, th)]
b = [r32.forward(x, w, th), r32.grad_input(gy, w, th), r32.grad_weight(gy, x, th)]
dev = torch.device("cuda:0")
ws = ConvWorkspace([LayerConfig(*key)])
xd, wd, gyd = (torch.from_numpy(t).to(dev) for t in (x, w, gy))
c = [ws.forward(xd, wd).cpu().numpy(), ws.grad_input(gyd, wd).cpu().numpy(), ws.grad_weight(gyd, xd).cpu().numpy()]
print(key, os.environ.get("FFTCONV_B200_SMALLSRC", "1"), os.environ.get("FFTCONV_B200_SMALLCROP", "1"),
      "ours:", ["%.2e" % oracle.rel_l2_error(cc, aa) for aa, cc in zip(a, c)],
      "ref fp32:", ["%.2e" % oracle.rel_l2_error(bb, aa) for aa, bb in zip(a, b)])
