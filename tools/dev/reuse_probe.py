"""Dev probe: reuse-across-layers bit stability (conv_fft_test.cpp:191-209)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig  # noqa: E402

a, b = LayerConfig(3, 6, 2, 3, 2), LayerConfig(5, 12, 3, 2, 1)
ws = ConvWorkspace([a, b], device=0)
rng = np.random.default_rng(0)
xa = rng.uniform(-1, 1, (2, 2, 6, 6)).astype(np.float32)
wa = rng.uniform(-1, 1, (3, 2, 3, 3)).astype(np.float32)
xb = rng.uniform(-1, 1, (1, 3, 12, 12)).astype(np.float32)
wb = rng.uniform(-1, 1, (2, 3, 5, 5)).astype(np.float32)
ref = oracle.forward_direct(xa.astype(np.float64), wa.astype(np.float64))
for trial in range(5):
    first = ws.forward(xa, wa)
    ws.forward(xb, wb)
    again = ws.forward(xa, wa)
    print(trial, 'first err', oracle.rel_l2_error(first, ref), 'again err', oracle.rel_l2_error(again, ref),
          'maxdiff', float(np.abs(first - again).max()), flush=True)
# device path too
d = torch.device('cuda:0')
xad, wad, xbd, wbd = (torch.from_numpy(v).to(d) for v in (xa, wa, xb, wb))
for trial in range(3):
    f1 = ws.forward(xad, wad).cpu().numpy()
    ws.forward(xbd, wbd)
    f2 = ws.forward(xad, wad).cpu().numpy()
    print('dev', trial, oracle.rel_l2_error(f1, ref), oracle.rel_l2_error(f2, ref), flush=True)
