"""CPU oracle for the FFT-convolution hot path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both loaded through ctypes:

* ``liboracle.so``  -- ``fftconv_oracle.c``, a plain-C restatement of the
  reference algorithm (fft.hpp:20-203, conv_fft.hpp:74-304,
  conv_direct.hpp:24-127, rng.hpp:21-47), in float64 and float32.
* ``_ref/libfftconv_ref.so`` -- the unmodified reference, compiled from its
  own headers by ``oracle/Makefile`` (``ref_shim.cpp`` only binds its API).
  It pins the restatement (tests/golden) and is the CPU baseline of
  bench.py.  It is git-ignored but travels to the GPU box prebuilt.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg import this package.  The product package ``paper_1312_5851_b200`` never
does.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfftconv_ref.so")

_sz = C.c_size_t
_u64 = C.c_uint64
_p = C.c_void_p

ROLE_INPUT, ROLE_WEIGHTS, ROLE_GRAD_OUTPUT = 1, 2, 3


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


def _dt(dtype):
    return "_f64" if np.dtype(dtype) == np.float64 else "_f32"


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle status {code} {what}")
        self.code = code


@lru_cache(maxsize=None)
def lib():
    if not os.path.exists(ORACLE_SO):
        raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
    L = C.CDLL(ORACLE_SO)
    L.orc_uniform_at.restype = C.c_double
    L.orc_uniform_at.argtypes = [_u64, _u64, _u64]
    L.orc_splitmix64.restype = _u64
    L.orc_splitmix64.argtypes = [_u64]
    L.orc_random_verify_configs.argtypes = [_sz, _u64, _p]
    for s in ("_f64", "_f32"):
        for name in ("orc_forward_fft", "orc_forward_direct", "orc_grad_weight_fft",
                     "orc_grad_weight_direct", "orc_grad_input_fft", "orc_grad_input_direct"):
            fn = getattr(L, name + s)
            fn.restype = C.c_int
            fn.argtypes = [_p, _p, _p, _sz, _sz, _sz, _sz, _sz]
        for name in ("orc_forward_direct_planes", "orc_grad_input_direct_planes",
                     "orc_grad_weight_direct_planes"):
            fn = getattr(L, name + s)
            fn.restype = C.c_int
            fn.argtypes = [_p, _p, _p, _sz, _sz, _sz, _sz, _sz, _p, _sz]
        getattr(L, "orc_r2c_plane" + s).argtypes = [_p, _sz, _sz, _sz, _p]
        getattr(L, "orc_c2r_plane" + s).argtypes = [_p, _sz, _p, _sz, _sz]
        getattr(L, "orc_fft_1d" + s).argtypes = [_p, _sz, C.c_int]
        getattr(L, "orc_fill_uniform" + s).argtypes = [_p, _sz, _u64, _u64, _u64]
    return L


def _chk(code):
    if code != 0:
        raise OracleError(code)


# ---------------------------------------------------------------- rng.hpp
def uniform_at(seed: int, role: int, index: int) -> float:
    return lib().orc_uniform_at(seed, role, index)


def fill_uniform(shape, seed: int, role: int, stream: int = 0, dtype=np.float32) -> np.ndarray:
    out = np.empty(shape, dtype=dtype)
    getattr(lib(), "orc_fill_uniform" + _dt(dtype))(_ptr(out), out.size, seed, role, stream)
    return out


def random_verify_configs(count: int, seed: int):
    out = np.zeros((count, 5), dtype=np.uint64)
    lib().orc_random_verify_configs(count, seed, _ptr(out))
    return [tuple(int(v) for v in row) for row in out]  # (k, n, f, f', S)


# ---------------------------------------------------------------- fft.hpp
def r2c_plane(src: np.ndarray, m: int) -> np.ndarray:
    src = np.ascontiguousarray(src)
    out = np.zeros((m, m // 2 + 1, 2), dtype=src.dtype)
    _chk(getattr(lib(), "orc_r2c_plane" + _dt(src.dtype))(_ptr(src), src.shape[0], src.shape[1], m, _ptr(out)))
    return out[..., 0] + 1j * out[..., 1]


def c2r_plane(half: np.ndarray, m: int, rows: int, cols: int, dtype=np.float64) -> np.ndarray:
    h = np.empty((m, m // 2 + 1, 2), dtype=dtype)
    h[..., 0], h[..., 1] = half.real, half.imag
    dst = np.zeros((rows, cols), dtype=dtype)
    _chk(getattr(lib(), "orc_c2r_plane" + _dt(dtype))(_ptr(h), m, _ptr(dst), rows, cols))
    return dst


def fft_1d(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    m = x.shape[0]
    d = np.empty((m, 2), dtype=np.float64)
    d[:, 0], d[:, 1] = x.real, x.imag
    _chk(lib().orc_fft_1d_f64(_ptr(d), m, int(inverse)))
    return d[:, 0] + 1j * d[:, 1]


# ------------------------------------------------------------ conv ops
def forward_fft(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    S, f, n, _ = x.shape
    fo, _, k, _ = w.shape
    y = np.zeros((S, fo, n - k + 1, n - k + 1), dtype=x.dtype)
    _chk(getattr(lib(), "orc_forward_fft" + _dt(x.dtype))(_ptr(x), _ptr(w), _ptr(y), S, f, fo, n, k))
    return y


def grad_input_fft(gy: np.ndarray, w: np.ndarray) -> np.ndarray:
    S, fo, no, _ = gy.shape
    _, f, k, _ = w.shape
    n = no + k - 1
    gx = np.zeros((S, f, n, n), dtype=gy.dtype)
    _chk(getattr(lib(), "orc_grad_input_fft" + _dt(gy.dtype))(_ptr(gy), _ptr(w), _ptr(gx), S, f, fo, no, k))
    return gx


def grad_weight_fft(gy: np.ndarray, x: np.ndarray) -> np.ndarray:
    S, fo, no, _ = gy.shape
    _, f, n, _ = x.shape
    k = n - no + 1
    gw = np.zeros((fo, f, k, k), dtype=x.dtype)
    _chk(getattr(lib(), "orc_grad_weight_fft" + _dt(x.dtype))(_ptr(gy), _ptr(x), _ptr(gw), S, f, fo, n, no))
    return gw


def forward_direct(x, w):
    S, f, n, _ = x.shape
    fo, _, k, _ = w.shape
    y = np.zeros((S, fo, n - k + 1, n - k + 1), dtype=x.dtype)
    _chk(getattr(lib(), "orc_forward_direct" + _dt(x.dtype))(_ptr(x), _ptr(w), _ptr(y), S, f, fo, n, k))
    return y


def grad_input_direct(gy, w):
    S, fo, no, _ = gy.shape
    _, f, k, _ = w.shape
    n = no + k - 1
    gx = np.zeros((S, f, n, n), dtype=gy.dtype)
    _chk(getattr(lib(), "orc_grad_input_direct" + _dt(gy.dtype))(_ptr(gy), _ptr(w), _ptr(gx), S, f, fo, no, k))
    return gx


def grad_weight_direct(gy, x):
    S, fo, no, _ = gy.shape
    _, f, n, _ = x.shape
    k = n - no + 1
    gw = np.zeros((fo, f, k, k), dtype=x.dtype)
    _chk(getattr(lib(), "orc_grad_weight_direct" + _dt(x.dtype))(_ptr(gy), _ptr(x), _ptr(gw), S, f, fo, n, no))
    return gw


def forward_direct_planes(x, w, plane_ids):
    """Selected (b*f'+o) planes of forward_direct, for layers too big for the full oracle."""
    S, f, n, _ = x.shape
    fo, _, k, _ = w.shape
    ids = np.ascontiguousarray(plane_ids, dtype=np.int64)
    out = np.zeros((len(ids), n - k + 1, n - k + 1), dtype=x.dtype)
    _chk(getattr(lib(), "orc_forward_direct_planes" + _dt(x.dtype))(
        _ptr(x), _ptr(w), _ptr(out), S, f, fo, n, k, _ptr(ids), len(ids)))
    return out


def grad_input_direct_planes(gy, w, plane_ids):
    """Selected (b*f+fi) planes of grad_input_direct."""
    S, fo, no, _ = gy.shape
    _, f, k, _ = w.shape
    n = no + k - 1
    ids = np.ascontiguousarray(plane_ids, dtype=np.int64)
    out = np.zeros((len(ids), n, n), dtype=gy.dtype)
    _chk(getattr(lib(), "orc_grad_input_direct_planes" + _dt(gy.dtype))(
        _ptr(gy), _ptr(w), _ptr(out), S, f, fo, no, k, _ptr(ids), len(ids)))
    return out


def grad_weight_direct_planes(gy, x, plane_ids):
    """Selected (o*f+fi) planes of grad_weight_direct."""
    S, fo, no, _ = gy.shape
    _, f, n, _ = x.shape
    k = n - no + 1
    ids = np.ascontiguousarray(plane_ids, dtype=np.int64)
    out = np.zeros((len(ids), k, k), dtype=x.dtype)
    _chk(getattr(lib(), "orc_grad_weight_direct_planes" + _dt(x.dtype))(
        _ptr(gy), _ptr(x), _ptr(out), S, f, fo, n, no, _ptr(ids), len(ids)))
    return out


# ------------------------------------------------------------ error norms
def max_rel_error(got: np.ndarray, ref: np.ndarray) -> float:
    """tensor.hpp:177-181: sup-norm error relative to the sup norm of ref."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref), initial=0.0) / max(np.max(np.abs(ref), initial=0.0), 1e-30))


def rel_l2_error(got: np.ndarray, ref: np.ndarray) -> float:
    """BASELINE.json bar: ||got - ref||_2 / ||ref||_2 <= 1e-4 (fp32)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


# ------------------------------------------------------------ reference
def ref_available() -> bool:
    return os.path.exists(REF_SO)


@lru_cache(maxsize=None)
def ref_lib():
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} missing: build it with `make -C oracle ref` where /root/reference exists")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_uniform_at.restype = C.c_double
    L.ref_uniform_at.argtypes = [_u64, _u64, _u64]
    L.ref_fill_uniform_f32.argtypes = [_p, _sz, _u64, _u64, _u64]
    L.ref_fill_uniform_f64.argtypes = [_p, _sz, _u64, _u64, _u64]
    L.ref_ws_create.argtypes = [_p, _sz, C.c_int, C.POINTER(_p)]
    L.ref_ws_destroy.argtypes = [_p]
    L.ref_ws_info.argtypes = [_p, _p]
    L.ref_ws_counters.argtypes = [_p, _p]
    L.ref_ws_reset_counters.argtypes = [_p]
    for s in ("_f32", "_f64"):
        getattr(L, "ref_ws_forward" + s).argtypes = [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, C.c_uint]
        getattr(L, "ref_ws_grad_input" + s).argtypes = [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _p, C.c_uint]
        getattr(L, "ref_ws_grad_weight" + s).argtypes = [_p, _p, _sz, _sz, _sz, _sz, _p, _sz, _sz, _sz, _sz, _p, C.c_uint]
        for name in ("ref_forward_direct", "ref_grad_input_direct", "ref_grad_weight_direct"):
            getattr(L, name + s).argtypes = [_p, _p, _p, _sz, _sz, _sz, _sz, _sz, C.c_uint]
        getattr(L, "ref_r2c_plane" + s).argtypes = [_p, _sz, _sz, _sz, _p]
        getattr(L, "ref_c2r_plane" + s).argtypes = [_p, _sz, _p, _sz, _sz]
    L.ref_fft_1d_f64.argtypes = [_p, _sz, C.c_int]
    L.ref_run_op_bench_f32.argtypes = [_sz, _sz, _sz, _sz, _sz, C.c_int, C.c_int, _sz, _sz, C.c_uint, _u64, _p]
    L.ref_resolve_threads.argtypes = [C.c_uint]
    L.ref_resolve_threads.restype = C.c_uint
    L.ref_random_verify_configs.argtypes = [_sz, _u64, _p]
    L.ref_run_iteration_f32.argtypes = [_p, _sz, _sz, _u64, C.c_int, C.c_uint, _p, _sz, C.POINTER(_sz), _p]
    L.ref_run_iteration_f64.argtypes = [_p, _sz, _sz, _u64, C.c_int, C.c_uint, _p, _sz, C.POINTER(_sz), _p]
    L.ref_cost_model.argtypes = [_sz, _sz, _sz, _sz, _sz, C.c_double, C.c_int, _p]
    return L


class RefWorkspace:
    """The reference ``fftconv::ConvWorkspace<T>`` driven through ref_shim.cpp."""

    def __init__(self, configs, dtype=np.float64):
        arr = np.ascontiguousarray(np.array(configs, dtype=np.uint64).reshape(-1, 5))
        h = _p()
        self.dtype = np.dtype(dtype)
        code = ref_lib().ref_ws_create(_ptr(arr), arr.shape[0], int(self.dtype == np.float64), C.byref(h))
        if code:
            raise OracleError(code, ref_lib().ref_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_ws_destroy(self.h)
            self.h = None

    def info(self):
        out = np.zeros(5, dtype=np.uint64)
        ref_lib().ref_ws_info(self.h, _ptr(out))
        return dict(zip(("max_fft_size", "capacity_x", "capacity_w", "capacity_y", "frequency_bytes"),
                        (int(v) for v in out)))

    def counters(self):
        out = np.zeros(3, dtype=np.uint64)
        ref_lib().ref_ws_counters(self.h, _ptr(out))
        return tuple(int(v) for v in out)

    def reset_counters(self):
        ref_lib().ref_ws_reset_counters(self.h)

    def _call(self, code):
        if code:
            raise OracleError(code, ref_lib().ref_last_error().decode())

    def forward(self, x, w, threads=1):
        x = np.ascontiguousarray(x, dtype=self.dtype)
        w = np.ascontiguousarray(w, dtype=self.dtype)
        S, f, r, c = x.shape
        fo, wi, k, _ = w.shape
        no = max(r - k + 1, 1)
        y = np.zeros((S, fo, no, no), dtype=self.dtype)
        self._call(getattr(ref_lib(), "ref_ws_forward" + _dt(self.dtype))(
            self.h, _ptr(x), S, f, r, c, _ptr(w), fo, wi, k, _ptr(y), threads))
        return y

    def grad_input(self, gy, w, threads=1):
        gy = np.ascontiguousarray(gy, dtype=self.dtype)
        w = np.ascontiguousarray(w, dtype=self.dtype)
        S, fo, r, c = gy.shape
        wo, f, k, _ = w.shape
        n = r + k - 1
        gx = np.zeros((S, f, n, n), dtype=self.dtype)
        self._call(getattr(ref_lib(), "ref_ws_grad_input" + _dt(self.dtype))(
            self.h, _ptr(gy), S, fo, r, c, _ptr(w), wo, f, k, _ptr(gx), threads))
        return gx

    def grad_weight(self, gy, x, threads=1):
        gy = np.ascontiguousarray(gy, dtype=self.dtype)
        x = np.ascontiguousarray(x, dtype=self.dtype)
        Sg, fo, r, c = gy.shape
        Sx, f, xr, xc = x.shape
        k = max(xr - r + 1, 1)
        gw = np.zeros((fo, f, k, k), dtype=self.dtype)
        self._call(getattr(ref_lib(), "ref_ws_grad_weight" + _dt(self.dtype))(
            self.h, _ptr(gy), Sg, fo, r, c, _ptr(x), Sx, f, xr, xc, _ptr(gw), threads))
        return gw


def ref_run_op_bench(k, n, f, fo, S, op, method, iters, warmup, threads, seed):
    """reference run_op_bench<float> (bench.hpp:80-145); returns dict of ms stats + checksum."""
    out = np.zeros(5, dtype=np.float64)
    code = ref_lib().ref_run_op_bench_f32(k, n, f, fo, S, op, method, iters, warmup, threads, seed, _ptr(out))
    if code:
        raise OracleError(code, ref_lib().ref_last_error().decode())
    return dict(zip(("mean_ms", "std_ms", "min_ms", "median_ms", "checksum"), (float(v) for v in out)))


def ref_run_iteration(stages, S: int, seed: int, engine: int = 1, threads: int = 0, dtype=np.float32):
    """reference run_iteration<float|double> (layers.hpp:441-609) on its own
    init_params / make_batch.  stages: records (kind, k, n, f, f'|fc outputs),
    kind 0 conv, 1 relu, 2 pool, 3 fc.  Returns (flat grads, scalars dict)."""
    L = ref_lib()
    fn = L.ref_run_iteration_f64 if np.dtype(dtype) == np.float64 else L.ref_run_iteration_f32
    rec = np.ascontiguousarray(np.asarray(stages, dtype=np.uint64).reshape(-1, 5))
    n = C.c_size_t(0)
    sc = np.zeros(6, dtype=np.float64)
    th = int(L.ref_resolve_threads(threads))
    code = fn(_ptr(rec), rec.shape[0], S, seed, engine, th, None, 0, C.byref(n), _ptr(sc))
    if code:
        raise OracleError(code, L.ref_last_error().decode())
    g = np.zeros(n.value, dtype=np.dtype(dtype))
    code = fn(_ptr(rec), rec.shape[0], S, seed, engine, th, _ptr(g), g.size, C.byref(n), _ptr(sc))
    if code:
        raise OracleError(code, L.ref_last_error().decode())
    keys = ("loss", "grad_checksum", "update_output_ms", "update_grad_input_ms", "acc_grad_ms",
            "grad_input_calls")
    return g, dict(zip(keys, (float(v) for v in sc)))


def ref_cost_model(k, n, f, fo, S, C, op):
    """cost_model.hpp ops_* (op 0 forward, 1 grad_input, 2 grad_weight) and
    memory_bytes / packed_memory_bytes(4)."""
    out = np.zeros(6, dtype=np.float64)
    code = ref_lib().ref_cost_model(k, n, f, fo, S, C, op, _ptr(out))
    if code:
        raise OracleError(code, ref_lib().ref_last_error().decode())
    return out
