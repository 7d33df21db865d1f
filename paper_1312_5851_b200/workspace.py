"""Python mirror of the reference operator interface, on the B200 kernels.

``ConvWorkspace`` follows fftconv::ConvWorkspace<T>
(/root/reference/proj/include/fftconv/conv_fft.hpp:40-312) method for method:
``forward(x, w, threads=1)``, ``grad_input(gy, w, threads=1)``,
``grad_weight(gy, x, threads=1)``, ``max_fft_size``, ``capacity_x/w/y``,
``frequency_bytes``, ``counters()``, ``reset_counters()``; the free functions
``workspace_for`` / ``forward_fft`` / ``grad_input_fft`` / ``grad_weight_fft``
mirror conv_fft.hpp:314-335.  Errors are the reference classes
(``errors.py``), raised in the reference's validation order.

Arguments may be
* CUDA ``torch.Tensor`` (fp32, contiguous): the device entry points run on
  the current stream, results stay in HBM; or
* ``numpy.ndarray`` (fp32): the host entry points copy in, compute on the
  GPU and copy the result back -- the drop-in for Tensor4/Weights4 storage.

There is no CPU path: every call goes through libfftconv_b200.so.
"""
from __future__ import annotations

import ctypes as C
from collections import namedtuple
from typing import Iterable, Sequence

import numpy as np

from . import _native
from .errors import ConfigError, raise_for_status
from .layer_config import LayerConfig

OpCounters = namedtuple("OpCounters", ["forward_transforms", "inverse_transforms", "complex_macs"])


def _is_torch(t) -> bool:
    return type(t).__module__.startswith("torch")


def _shape4(t):
    s = tuple(int(v) for v in t.shape)
    if len(s) != 4:
        raise ValueError(f"expected a rank-4 tensor, got shape {s}")
    return s


def _weights_shape(t):
    s = _shape4(t)
    if s[2] != s[3]:
        # Weights4 kernels are square by construction (tensor.hpp:65-108).
        raise ValueError(f"Weights4 kernels must be square, got {s}")
    return s[0], s[1], s[2]


class ConvWorkspace:
    """B200 drop-in for ``fftconv::ConvWorkspace<float>``."""

    def __init__(self, configs: Sequence, device: int | None = None):
        cfgs = [c if isinstance(c, LayerConfig) else LayerConfig(*c) for c in configs]
        if device is None:
            device = 0
            try:
                import torch

                if torch.cuda.is_available():
                    device = torch.cuda.current_device()
            except ImportError:
                pass
        self.device = int(device)
        L = _native.lib()
        arr = (_native.Layer * max(len(cfgs), 1))()
        for i, c in enumerate(cfgs):
            arr[i] = _native.Layer(c.kernel, c.image, c.in_maps, c.out_maps, c.batch)
        h = C.c_void_p()
        code = L.fftconv_b200_ws_create(arr, len(cfgs), self.device, C.byref(h))
        raise_for_status(code, _native.last_error(None))
        self._h = h
        self.configs = cfgs

    def close(self):
        if getattr(self, "_h", None):
            _native.lib().fftconv_b200_ws_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------- introspection
    def _info(self):
        out = (C.c_uint64 * 6)()
        _native.lib().fftconv_b200_ws_info(self._h, out)
        return list(out)

    def max_fft_size(self) -> int:
        return int(self._info()[0])

    def capacity_x(self) -> int:
        return int(self._info()[1])

    def capacity_w(self) -> int:
        return int(self._info()[2])

    def capacity_y(self) -> int:
        return int(self._info()[3])

    def frequency_bytes(self) -> int:
        """Reference accounting (cap_x+cap_w+cap_y)*sizeof(complex<float>), conv_fft.hpp:66-69."""
        return int(self._info()[4])

    def device_bytes(self) -> int:
        """Bytes of HBM the B200 workspace actually holds (padded GEMM layouts)."""
        return int(self._info()[5])

    def counters(self) -> OpCounters:
        out = (C.c_uint64 * 3)()
        _native.lib().fftconv_b200_counters(self._h, out)
        return OpCounters(*(int(v) for v in out))

    def reset_counters(self) -> None:
        _native.lib().fftconv_b200_reset_counters(self._h)

    def set_stage_timing(self, enable: bool) -> None:
        _native.lib().fftconv_b200_set_stage_timing(self._h, int(bool(enable)))

    def stage_ms(self):
        out = (C.c_float * 4)()
        code = _native.lib().fftconv_b200_stage_ms(self._h, out)
        raise_for_status(code, _native.last_error(self._h))
        return [float(v) for v in out]

    def set_span_timing(self, enable: bool) -> None:
        """Live per-kernel spans with the PDL chain intact (include/fftconv_b200.h)."""
        code = _native.lib().fftconv_b200_set_span_timing(self._h, int(bool(enable)))
        raise_for_status(code, _native.last_error(self._h))

    def span_ms(self, max_ops: int = 128):
        """[(k1_ms, gemm_ms, k4_ms)] per operator since set_span_timing(True); None where not recorded."""
        out = (C.c_float * (3 * max_ops))()
        n = int(_native.lib().fftconv_b200_span_ms(self._h, out, max_ops))
        if n < 0:
            raise_for_status(-n, _native.last_error(self._h))
        return [tuple(None if out[3 * i + k] < 0 else float(out[3 * i + k]) for k in range(3)) for i in range(n)]

    def last_gemm_path(self) -> str | None:
        """Which GEMM kernel ran in the last call: "f16x3", "tf32x3" or None
        (synchronises the device; include/fftconv_b200.h)."""
        v = int(_native.lib().fftconv_b200_last_gemm_path(self._h))
        return {1: "f16x3", 0: "tf32x3"}.get(v)

    def set_gemm_kind(self, kind: str | None) -> str | None:
        """This workspace's K3 precision scheme ("tf32x3", "f16x3", "auto"), or
        None for the process default; returns the previous override."""
        code = -1 if kind is None else _native.GEMM_KINDS[kind]
        prev = int(_native.lib().fftconv_b200_ws_set_gemm_kind(self._h, code))
        return {v: k for k, v in _native.GEMM_KINDS.items()}.get(prev)

    def last_launch_count(self) -> int:
        return int(_native.lib().fftconv_b200_last_launch_count(self._h))

    # ---------------------------------------------------------- operators
    def _check(self, code):
        raise_for_status(code, _native.last_error(self._h))

    @staticmethod
    def _stream(t):
        import torch

        return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)

    @staticmethod
    def _dev_ptr(t):
        import torch

        if t.dtype != torch.float32 or not t.is_cuda:
            raise TypeError("device operands must be CUDA float32 tensors")
        if not t.is_contiguous():
            raise ValueError("device operands must be contiguous")
        return C.c_void_p(t.data_ptr())

    @staticmethod
    def _host(a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        return a, a.ctypes.data_as(C.c_void_p)

    @staticmethod
    def _host_out(out, shape):
        """Result buffer for the host path: `out` (e.g. pinned) when given."""
        if out is None:
            return np.zeros(shape, dtype=np.float32)
        if out.shape != tuple(shape) or out.dtype != np.float32 or not out.flags.c_contiguous:
            raise ValueError(f"out must be a C-contiguous float32 array of shape {tuple(shape)}")
        return out

    def forward(self, x, w, threads: int = 1, out=None, relu: bool = False, image: int | None = None):
        """conv_fft.hpp:74-113: y = valid cross-correlation of x by w.
        Device-operand extensions for the layer stack: relu=True fuses the
        following relu (layers.hpp:88-97) into the inverse transform's
        stores; image > x's planes treats x as the top-left of an image x
        image layer input, zeros elsewhere (fit_to's pad, folded in)."""
        S, f, xr, xc = _shape4(x)
        wo, wi, k = _weights_shape(w)
        n = image if image else xr
        no = n - k + 1 if k <= n else 1
        L = _native.lib()
        if _is_torch(x):
            import torch

            y = torch.empty((S, wo, max(no, 1), max(no, 1)), dtype=torch.float32, device=x.device)
            if image and image != xr:
                code = L.fftconv_b200_forward_fit(self._h, self._dev_ptr(x), S, f, xr, xc, int(image),
                                                  self._dev_ptr(w), wo, wi, k, self._dev_ptr(y), 1 if relu else 0,
                                                  self._stream(x))
            else:
                fn = L.fftconv_b200_forward_relu if relu else L.fftconv_b200_forward
                code = fn(self._h, self._dev_ptr(x), S, f, xr, xc, self._dev_ptr(w), wo, wi, k, self._dev_ptr(y),
                          self._stream(x))
            self._check(code)
            return y
        if relu or image:
            raise ValueError("forward(relu=..., image=...) take device operands")
        xa, xp = self._host(x)
        wa, wp = self._host(w)
        y = self._host_out(out, (S, wo, max(no, 1), max(no, 1)))
        code = L.fftconv_b200_forward_host(self._h, xp, S, f, xr, xc, wp, wo, wi, k,
                                           y.ctypes.data_as(C.c_void_p), int(threads))
        self._check(code)
        return y

    def grad_input(self, gy, w, threads: int = 1, out=None, size: int | None = None):
        """conv_fft.hpp:115-152: gx = full convolution of gy by w.  size
        (device operands): only the top-left size x size of each plane
        (fit_to's crop back to a pre-pad input, folded in)."""
        S, fo, gr, gc = _shape4(gy)
        wo, wi, k = _weights_shape(w)
        n = gr + k - 1
        L = _native.lib()
        if _is_torch(gy):
            import torch

            if size and size != n:
                gx = torch.empty((S, wi, size, size), dtype=torch.float32, device=gy.device)
                code = L.fftconv_b200_grad_input_fit(self._h, self._dev_ptr(gy), S, fo, gr, gc, self._dev_ptr(w),
                                                     wo, wi, k, self._dev_ptr(gx), int(size), self._stream(gy))
            else:
                gx = torch.empty((S, wi, n, n), dtype=torch.float32, device=gy.device)
                code = L.fftconv_b200_grad_input(self._h, self._dev_ptr(gy), S, fo, gr, gc, self._dev_ptr(w), wo,
                                                 wi, k, self._dev_ptr(gx), self._stream(gy))
            self._check(code)
            return gx
        if size:
            raise ValueError("grad_input(size=...) takes device operands")
        ga, gp = self._host(gy)
        wa, wp = self._host(w)
        gx = self._host_out(out, (S, wi, n, n))
        code = L.fftconv_b200_grad_input_host(self._h, gp, S, fo, gr, gc, wp, wo, wi, k,
                                              gx.ctypes.data_as(C.c_void_p), int(threads))
        self._check(code)
        return gx

    def grad_weight(self, gy, x, threads: int = 1, out=None, image: int | None = None):
        """conv_fft.hpp:154-206: gw = batch-summed valid correlation of x by gy.
        image (device operands): x as in forward(image=...)."""
        Sg, fo, gr, gc = _shape4(gy)
        Sx, f, xr, xc = _shape4(x)
        n = image if image else xr
        k = n - gr + 1 if gr <= n else 1
        L = _native.lib()
        if _is_torch(gy):
            import torch

            gw = torch.empty((fo, f, k, k), dtype=torch.float32, device=gy.device)
            if image and image != xr:
                code = L.fftconv_b200_grad_weight_fit(self._h, self._dev_ptr(gy), Sg, fo, gr, gc, self._dev_ptr(x),
                                                      Sx, f, xr, xc, int(image), self._dev_ptr(gw),
                                                      self._stream(gy))
            else:
                code = L.fftconv_b200_grad_weight(self._h, self._dev_ptr(gy), Sg, fo, gr, gc, self._dev_ptr(x), Sx,
                                                  f, xr, xc, self._dev_ptr(gw), self._stream(gy))
            self._check(code)
            return gw
        if image:
            raise ValueError("grad_weight(image=...) takes device operands")
        ga, gp = self._host(gy)
        xa, xp = self._host(x)
        gw = self._host_out(out, (fo, f, k, k))
        code = L.fftconv_b200_grad_weight_host(self._h, gp, Sg, fo, gr, gc, xp, Sx, f, xr, xc,
                                               gw.ctypes.data_as(C.c_void_p), int(threads))
        self._check(code)
        return gw


def workspace_for(configs: Iterable, device: int | None = None) -> ConvWorkspace:
    """conv_fft.hpp:314-317"""
    cfgs = list(configs)
    if not cfgs:
        raise ConfigError("workspace: at least one layer config required")
    return ConvWorkspace(cfgs, device)


def forward_fft(ws: ConvWorkspace, x, w, threads: int = 1):
    """conv_fft.hpp:319-323"""
    return ws.forward(x, w, threads)


def grad_input_fft(ws: ConvWorkspace, gy, w, threads: int = 1):
    """conv_fft.hpp:325-329"""
    return ws.grad_input(gy, w, threads)


def grad_weight_fft(ws: ConvWorkspace, gy, x, threads: int = 1):
    """conv_fft.hpp:331-335"""
    return ws.grad_weight(gy, x, threads)
