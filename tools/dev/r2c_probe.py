"""Dev probe: r2c of an impulse / ramp at small m, printed."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_1312_5851_b200 import kernels  # noqa: E402

np.set_printoptions(precision=3, suppress=True, linewidth=150)
for m in (4, 8):
    x = np.zeros((1, m, m), dtype=np.float32)
    x[0, 0, 0] = 1
    print('impulse m', m)
    print(kernels.r2c(torch.from_numpy(x).cuda(), m).cpu().numpy()[0])
    x = np.arange(m * m, dtype=np.float32).reshape(1, m, m) / 10
    got = kernels.r2c(torch.from_numpy(x).cuda(), m).cpu().numpy()[0]
    ref = np.fft.fft2(x[0])[: m // 2 + 1]
    print('ramp got\n', got, '\nref\n', ref)
