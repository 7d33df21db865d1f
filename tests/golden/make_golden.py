"""Generates tests/golden/reference_golden.npz from the REFERENCE itself.

Runs the unmodified reference library (compiled from /root/reference headers
into oracle/_ref/libfftconv_ref.so by oracle/Makefile) on seeded inputs and
records inputs + outputs.  tests/test_oracle_golden.py pins the C oracle
restatement against these vectors, so the oracle used by every GPU parity
test is anchored to the reference's actual behaviour.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import RefWorkspace, ref_lib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")

# (k, n, f, f', S, seed): conv_fft_test.cpp shapes, non-pow2 n (m > n), the
# tight m == n case, m = 1/2, and BASELINE configs[0].
CASES = [
    (3, 16, 4, 6, 2, 11), (5, 16, 4, 4, 2, 12), (7, 32, 3, 5, 1, 13), (1, 7, 2, 3, 2, 14),
    (4, 9, 1, 1, 3, 15), (3, 8, 2, 2, 2, 31), (8, 8, 1, 2, 1, 32), (1, 1, 1, 2, 1, 33),
    (2, 2, 2, 1, 2, 34), (11, 20, 3, 2, 2, 35), (5, 32, 16, 16, 8, 1234),
]


def ref_fill(shape, seed, role, dtype):
    out = np.empty(shape, dtype=dtype)
    fn = ref_lib().ref_fill_uniform_f64 if dtype == np.float64 else ref_lib().ref_fill_uniform_f32
    fn(out.ctypes.data_as(oracle._p), out.size, seed, role, 0)
    return out


def ref_direct(name, *arrs, dims):
    out_shape, args = dims
    out = np.zeros(out_shape, dtype=np.float64)
    fn = getattr(ref_lib(), name + "_f64")
    code = fn(*(a.ctypes.data_as(oracle._p) for a in arrs), out.ctypes.data_as(oracle._p), *args, 1)
    assert code == 0
    return out


def main():
    if not oracle.ref_available():
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    data = {}
    for idx, (k, n, f, fo, S, seed) in enumerate(CASES):
        no = n - k + 1
        pre = f"c{idx}_"
        data[pre + "cfg"] = np.array([k, n, f, fo, S, seed], dtype=np.int64)
        big = S * f * n * n > 50000
        for dt, tag in (((np.float32, "f32"),) if big else ((np.float64, "f64"), (np.float32, "f32"))):
            x = ref_fill((S, f, n, n), seed, 1, dt)
            w = ref_fill((fo, f, k, k), seed, 2, dt)
            gy = ref_fill((S, fo, no, no), seed, 3, dt)
            ws = RefWorkspace([(k, n, f, fo, S)], dtype=dt)
            data[pre + f"x_{tag}"] = x
            data[pre + f"w_{tag}"] = w
            data[pre + f"gy_{tag}"] = gy
            data[pre + f"y_fft_{tag}"] = ws.forward(x, w)
            data[pre + f"gx_fft_{tag}"] = ws.grad_input(gy, w)
            data[pre + f"gw_fft_{tag}"] = ws.grad_weight(gy, x)
            data[pre + f"counters_{tag}"] = np.array(ws.counters(), dtype=np.uint64)
            if tag == "f64":
                data[pre + "y_direct_f64"] = ref_direct("ref_forward_direct", x, w,
                                                        dims=((S, fo, no, no), (S, f, fo, n, k)))
                data[pre + "gx_direct_f64"] = ref_direct("ref_grad_input_direct", gy, w,
                                                         dims=((S, f, n, n), (S, f, fo, no, k)))
                data[pre + "gw_direct_f64"] = ref_direct("ref_grad_weight_direct", gy, x,
                                                         dims=((fo, f, k, k), (S, f, fo, n, no)))
    # single-plane transforms (fft.hpp:160-203) at every supported m
    for m in (1, 2, 4, 8, 16, 32, 64):
        for src in sorted({1, max(1, m // 2 + 1), m}):
            if src > m:
                continue
            plane = ref_fill((src, src), 500 + m + src, 1, np.float64)
            half = np.zeros((m, m // 2 + 1, 2))
            assert ref_lib().ref_r2c_plane_f64(plane.ctypes.data_as(oracle._p), src, src, m,
                                               half.ctypes.data_as(oracle._p)) == 0
            data[f"r2c_m{m}_s{src}_in"] = plane
            data[f"r2c_m{m}_s{src}_out"] = half
            back = np.zeros((src, src))
            assert ref_lib().ref_c2r_plane_f64(half.ctypes.data_as(oracle._p), m,
                                               back.ctypes.data_as(oracle._p), src, src) == 0
            data[f"c2r_m{m}_s{src}_out"] = back
    # rng known answers (rng.hpp) and the verify-sweep draws (bench.hpp:164-183)
    data["uniform_at_1234_1"] = np.array([ref_lib().ref_uniform_at(1234, 1, i) for i in range(16)])
    cfgs = np.zeros((100, 5), dtype=np.uint64)
    ref_lib().ref_random_verify_configs(100, 2024, cfgs.ctypes.data_as(oracle._p))
    data["verify_configs_2024"] = cfgs
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT} ({os.path.getsize(OUT) / 1e6:.2f} MB, {len(data)} arrays)")


if __name__ == "__main__":
    main()
