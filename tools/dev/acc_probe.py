"""Accuracy breakdown at P: each operator vs fp64 (reference ConvWorkspace<double>),
the reference's own fp32 path beside it, and K1 / K3 / K4 alone vs fp64 numpy."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig, kernels  # noqa: E402

dev = torch.device("cuda:0")
key = (7, 32, 96, 96, 128)
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
for kind in ("tf32x3", "f16x3"):
    ws = ConvWorkspace([LayerConfig(*key)])
    ws.set_gemm_kind(kind)
    xd, wd, gyd = (torch.from_numpy(t).to(dev) for t in (x, w, gy))
    c = [ws.forward(xd, wd).cpu().numpy(), ws.grad_input(gyd, wd).cpu().numpy(), ws.grad_weight(gyd, xd).cpu().numpy()]
    print(kind, "ours vs fp64:", ["%.2e" % oracle.rel_l2_error(cc, aa) for aa, cc in zip(a, c)],
          " ref fp32 vs fp64:", ["%.2e" % oracle.rel_l2_error(bb, aa) for aa, bb in zip(a, b)])
# K1 alone
planes = torch.from_numpy(x[:4].reshape(-1, n, n).copy()).to(dev)
spec = kernels.r2c(planes, 32).cpu().numpy()
ref = np.fft.fft2(x[:4].reshape(-1, n, n).astype(np.float64), s=(32, 32))[:, :17, :]
print("K1 r2c vs fp64:", "%.2e" % (np.linalg.norm(spec.reshape(ref.shape) - ref) / np.linalg.norm(ref)))
# K4 alone
P = np.fft.fft2(np.random.default_rng(0).standard_normal((64, 32, 32)))[:, :17, :]
out = kernels.c2r(torch.from_numpy(P.astype(np.complex64)).to(dev), 26).cpu().numpy()
refo = np.fft.ifft2(np.concatenate([P, np.conj(P[:, 15:0:-1, :][:, :, (-np.arange(32)) % 32])], axis=1)).real[:, :26, :26]
print("K4 c2r vs fp64:", "%.2e" % (np.linalg.norm(out - refo) / np.linalg.norm(refo)))
# K3 alone
rng = np.random.default_rng(1)
A = (rng.standard_normal((8, 128, 96)) + 1j * rng.standard_normal((8, 128, 96)))
B = (rng.standard_normal((8, 96, 96)) + 1j * rng.standard_normal((8, 96, 96)))
for kind in ("tf32x3", "f16x3"):
    from paper_1312_5851_b200 import _native
    prev = _native.set_gemm_kind(kind)
    D = kernels.cgemm(torch.from_numpy(A.astype(np.complex64)).to(dev), torch.from_numpy(B.astype(np.complex64)).to(dev), 0).cpu().numpy()
    _native.set_gemm_kind(prev)
    Dr = np.einsum("tmk,tnk->tnm", A.astype(np.complex64).astype(np.complex128), np.conj(B.astype(np.complex64).astype(np.complex128)))
    Df = np.einsum("tmk,tnk->tnm", A.astype(np.complex64), np.conj(B.astype(np.complex64)))
    print(kind, "K3 vs fp64:", "%.2e" % (np.linalg.norm(D - Dr) / np.linalg.norm(Dr)),
          " numpy complex64 einsum vs fp64: %.2e" % (np.linalg.norm(Df - Dr) / np.linalg.norm(Dr)))
