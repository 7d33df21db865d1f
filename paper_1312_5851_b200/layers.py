"""Training-step driver over the B200 convolution operators.

Mirror of the reference layer stack (/root/reference/proj/include/fftconv/
layers.hpp): the network grammar (`conv k n f fp`, `relu`, `pool`,
`fc outputs`; :250-311), the presets (:321-348), parameter and batch
generation (:355-390), `fit_to` (:393-407) and `run_iteration` (:441-609):
forward through all stages, loss = sum of the final outputs, backward
collecting every weight gradient, the first conv layer skipping its
grad-input pass.

Everything runs on the GPU: the conv stages through the B200
ConvWorkspace (fprop / bprop / accGrad kernels), relu / max-pool / fit_to
through the library's layer-stack kernels (csrc/layers.cuh), and the final
fully connected layer as a plain fp32 cuBLAS GEMM (TF32 disabled) through
torch.  Times are CUDA-event device times per reference category
(updateOutput / updateGradInput / accGradParameters).
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native
from .errors import ConfigError, ShapeError, raise_for_status
from .layer_config import LayerConfig
from .rng import ROLE_INPUT, ROLE_WEIGHTS, fill_uniform
from .workspace import ConvWorkspace

ROLE_FC_WEIGHTS = 4  # rng.hpp:15-16
ROLE_FC_BIAS = 5


class StageKind(enum.IntEnum):  # layers.hpp:182
    conv = 0
    relu = 1
    pool = 2
    fc = 3


@dataclass
class Stage:  # layers.hpp:184-189
    kind: StageKind = StageKind.relu
    conv: Optional[LayerConfig] = None
    fc_outputs: int = 0

    def record(self):
        """(kind, k, n, f, f' | fc outputs): the oracle shim's stage record."""
        if self.kind == StageKind.conv:
            c = self.conv
            return (int(self.kind), c.kernel, c.image, c.in_maps, c.out_maps)
        return (int(self.kind), 0, 0, 0, self.fc_outputs)


@dataclass
class NetShape:  # layers.hpp:192-197
    conv_count: int = 0
    final_maps: int = 0
    final_size: int = 0
    has_fc: bool = False
    fc_inputs: int = 0
    fc_outputs: int = 0


@dataclass
class NetworkSpec:  # layers.hpp:199-249
    stages: List[Stage] = field(default_factory=list)
    input_maps: int = 0
    input_image: int = 0
    default_batch: int = 1

    def shape(self) -> NetShape:
        """Walks the stages checking map chaining, pooling parity and fc
        placement (layers.hpp:207-246)."""
        if not self.stages:
            raise ConfigError("network: no stages")
        if self.stages[0].kind != StageKind.conv:
            raise ConfigError("network: first stage must be a convolution")
        out = NetShape()
        maps = self.stages[0].conv.in_maps
        size = 0
        first = True
        for st in self.stages:
            if out.has_fc:
                raise ConfigError("network: fc must be the last stage")
            if st.kind == StageKind.conv:
                c = LayerConfig(st.conv.kernel, st.conv.image, st.conv.in_maps, st.conv.out_maps, 1)
                c.validate()
                if not first and c.in_maps != maps:
                    raise ConfigError(f"network: conv expects {c.in_maps} maps but gets {maps}")
                maps = c.out_maps
                size = c.output_size()
                first = False
                out.conv_count += 1
            elif st.kind == StageKind.pool:
                if size % 2 != 0:
                    raise ConfigError(f"network: pool needs an even plane size, got {size}")
                size //= 2
            elif st.kind == StageKind.fc:
                if st.fc_outputs == 0:
                    raise ConfigError("network: fc outputs must be >= 1")
                out.has_fc = True
                out.fc_inputs = maps * size * size
                out.fc_outputs = st.fc_outputs
        out.final_maps = maps
        out.final_size = size
        return out

    def validate(self) -> None:
        self.shape()

    def conv_configs(self, batch: int) -> List[LayerConfig]:
        return [LayerConfig(s.conv.kernel, s.conv.image, s.conv.in_maps, s.conv.out_maps, batch)
                for s in self.stages if s.kind == StageKind.conv]

    def records(self):
        return [s.record() for s in self.stages]


def parse_network(text: str) -> NetworkSpec:
    """One stage per line: `conv k n f fp`, `relu`, `pool`, `fc outputs`;
    blank lines and text after # ignored (layers.hpp:250-304)."""
    spec = NetworkSpec()
    for line_no, raw in enumerate(text.splitlines(), 1):
        raw = raw.split("#", 1)[0]
        words = raw.split()
        if not words:
            continue
        word, rest = words[0], words[1:]

        def want(what, _rest=rest):
            if not _rest:
                raise ConfigError(f"network file line {line_no}: expected positive {what}")
            tok = _rest.pop(0)
            try:
                v = int(tok)
            except ValueError:
                raise ConfigError(f"network file line {line_no}: expected positive {what}") from None
            if v < 1:
                raise ConfigError(f"network file line {line_no}: expected positive {what}")
            return v

        if word == "conv":
            st = Stage(StageKind.conv, LayerConfig(want("kernel size"), want("image size"),
                                                   want("input map count"), want("output map count"), 1))
        elif word == "relu":
            st = Stage(StageKind.relu)
        elif word == "pool":
            st = Stage(StageKind.pool)
        elif word == "fc":
            st = Stage(StageKind.fc, fc_outputs=want("output count"))
        else:
            raise ConfigError(f"network file line {line_no}: unknown stage '{word}'")
        if rest:
            raise ConfigError(f"network file line {line_no}: unexpected token '{rest[0]}'")
        spec.stages.append(st)
    if not spec.stages:
        raise ConfigError("network file: no stages")
    if spec.stages[0].kind == StageKind.conv:
        spec.input_maps = spec.stages[0].conv.in_maps
        spec.input_image = spec.stages[0].conv.image
    spec.validate()
    return spec


PRESETS = {  # layers.hpp:321-348
    "reference-net": (128, "conv 11 32 3 96\nrelu\nconv 7 32 96 256\nrelu\npool\nconv 5 16 256 384\nrelu\n"
                           "conv 5 16 384 384\nrelu\nconv 3 16 384 384\nrelu\npool\nfc 1000\n"),
    # BASELINE configs[4] ("AlexNet-style 5-conv-layer stack, first layer
    # f = 3 -> 96, n = 128") in the reference grammar: AlexNet's map counts
    # and kernel sizes, fit_to between layers as in the reference preset
    "alexnet-128": (128, "conv 11 128 3 96\nrelu\npool\nconv 5 64 96 256\nrelu\npool\nconv 3 32 256 384\nrelu\n"
                         "conv 3 32 384 384\nrelu\nconv 3 32 384 256\nrelu\npool\nfc 1000\n"),
    "reference-net-small": (8, "conv 11 32 3 12\nrelu\nconv 7 32 12 32\nrelu\npool\nconv 5 16 32 48\nrelu\n"
                               "conv 5 16 48 48\nrelu\nconv 3 16 48 48\nrelu\npool\nfc 1000\n"),
}


def preset_network(name: str) -> NetworkSpec:
    if name not in PRESETS:
        raise ConfigError(f"unknown preset '{name}'")
    batch, text = PRESETS[name]
    spec = parse_network(text)
    spec.default_batch = batch
    return spec


@dataclass
class NetworkParams:  # layers.hpp:355-383 (host fp32 arrays)
    conv: List[np.ndarray]
    fc_weights: Optional[np.ndarray] = None  # outputs x inputs
    fc_bias: Optional[np.ndarray] = None


def init_params(spec: NetworkSpec, seed: int) -> NetworkParams:
    sh = spec.shape()
    conv = []
    for ci, c in enumerate(spec.conv_configs(1)):
        conv.append(fill_uniform((c.out_maps, c.in_maps, c.kernel, c.kernel), seed, ROLE_WEIGHTS, stream=ci))
    p = NetworkParams(conv)
    if sh.has_fc:
        p.fc_weights = fill_uniform((sh.fc_outputs, sh.fc_inputs), seed, ROLE_FC_WEIGHTS)
        p.fc_bias = fill_uniform((sh.fc_outputs,), seed, ROLE_FC_BIAS)
    return p


def make_batch(spec: NetworkSpec, S: int, seed: int) -> np.ndarray:  # layers.hpp:385-390
    return fill_uniform((S, spec.input_maps, spec.input_image, spec.input_image), seed, ROLE_INPUT)


@dataclass
class StageTimes:  # layers.hpp:414-424
    update_output_ms: float = 0.0
    update_grad_input_ms: float = 0.0
    acc_grad_ms: float = 0.0

    def total_ms(self) -> float:
        return self.update_output_ms + self.update_grad_input_ms + self.acc_grad_ms


@dataclass
class IterationResult:  # layers.hpp:426-437
    times: StageTimes
    loss: float
    conv_weight_grads: list       # device tensors [f'][f][k][k]
    fc_weight_grad: object = None
    fc_bias_grad: object = None
    grad_input_calls: int = 0
    grad_checksum: float = 0.0
    gpu_launches: int = 0           # our kernels (conv operators + layer stages; fc is cuBLAS)


# ---------------------------------------------------------------- device stages
_LAUNCHES = [0]  # our kernel launches since the last reset (run_iteration reports them)


def _launched(n: int = 1) -> None:
    _LAUNCHES[0] += n


class _CountingWorkspace:
    """Forwards the three operators and adds each call's launch count."""

    def __init__(self, ws):
        self.ws = ws

    def _run(self, fn, *a):
        r = fn(*a)
        _launched(self.ws.last_launch_count())
        return r

    def forward(self, x, w, relu=False, image=None):
        if relu or image:
            return self._run(lambda a, b: self.ws.forward(a, b, relu=relu, image=image), x, w)
        return self._run(self.ws.forward, x, w)

    def grad_input(self, gy, w, size=None):
        if size:
            return self._run(lambda a, b: self.ws.grad_input(a, b, size=size), gy, w)
        return self._run(self.ws.grad_input, gy, w)

    def grad_weight(self, gy, x, image=None):
        if image:
            return self._run(lambda a, b: self.ws.grad_weight(a, b, image=image), gy, x)
        return self._run(self.ws.grad_weight, gy, x)


def _stream_ptr(torch):
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def fit_to(t, size: int):
    """Pads (zeros) or crops every plane at the top-left to size x size
    (layers.hpp:393-407); returns t itself when it already fits."""
    import torch

    S, M, R, Cc = t.shape
    if R == size and Cc == size:
        return t
    out = torch.empty((S, M, size, size), dtype=torch.float32, device=t.device)
    raise_for_status(_native.lib().fftconv_b200_fit_to(_ptr(t), S * M, R, Cc, _ptr(out), size,
                                                        _stream_ptr(torch)), _native.last_error(None))
    _launched()
    return out


def relu_forward(x):
    import torch

    y = torch.empty_like(x)
    raise_for_status(_native.lib().fftconv_b200_relu_forward(_ptr(x), _ptr(y), x.numel(), _stream_ptr(torch)),
                     _native.last_error(None))
    _launched()
    return y


def relu_backward(gy, x):
    import torch

    if tuple(gy.shape) != tuple(x.shape):
        raise ShapeError("relu backward: gradient shape mismatch")
    gx = torch.empty_like(x)
    raise_for_status(_native.lib().fftconv_b200_relu_backward(_ptr(gy), _ptr(x), _ptr(gx), x.numel(),
                                                               _stream_ptr(torch)), _native.last_error(None))
    _launched()
    return gx


def maxpool_forward(x):
    """Returns (y, argmax, input shape) (layers.hpp:34-66)."""
    import torch

    S, M, R, Cc = x.shape
    y = torch.empty((S, M, R // 2, Cc // 2), dtype=torch.float32, device=x.device)
    arg = torch.empty((S, M, R // 2, Cc // 2), dtype=torch.int32, device=x.device)
    raise_for_status(_native.lib().fftconv_b200_maxpool_forward(_ptr(x), S * M, R, Cc, _ptr(y), _ptr(arg),
                                                                 _stream_ptr(torch)), _native.last_error(None))
    _launched()
    return y, arg, (S, M, R, Cc)


def maxpool_backward(gy, rec):
    import torch

    y, arg, shape = rec
    if tuple(gy.shape) != tuple(y.shape):
        raise ShapeError("maxpool backward: gradient shape mismatch")
    S, M, R, Cc = shape
    gx = torch.empty(shape, dtype=torch.float32, device=gy.device)
    raise_for_status(_native.lib().fftconv_b200_maxpool_backward(_ptr(gy), _ptr(arg), S * M, R, Cc, _ptr(gx),
                                                                  _stream_ptr(torch)), _native.last_error(None))
    _launched()
    return gx


def maxpool_relu_backward(gy, rec):
    """maxpool_backward then the backward of the relu that fed the pool, in
    one pass (fftconv_b200_maxpool_relu_backward): the relu mask at a
    window's winner is the pooled value > 0."""
    import torch

    y, arg, shape = rec
    if tuple(gy.shape) != tuple(y.shape):
        raise ShapeError("maxpool backward: gradient shape mismatch")
    S, M, R, Cc = shape
    gx = torch.empty(shape, dtype=torch.float32, device=gy.device)
    raise_for_status(_native.lib().fftconv_b200_maxpool_relu_backward(_ptr(gy), _ptr(arg), _ptr(y), S * M, R, Cc,
                                                                       _ptr(gx), _stream_ptr(torch)),
                     _native.last_error(None))
    _launched()
    return gx


def run_iteration(spec: NetworkSpec, params: NetworkParams, batch, ws: ConvWorkspace | None = None,
                  device: int = 0, group=None, comm=None, chunks: int = 4) -> IterationResult:
    """One training iteration (layers.hpp:441-609) on the GPU.  `batch` is a
    host array or a CUDA tensor [S][maps][n][n]; parameters are host arrays
    (copied to the device once per call, outside the timed categories).

    Data-parallel (BASELINE configs[4] on N GPUs): with torch.distributed
    initialised and more than one rank in `group`, `batch` is this rank's
    minibatch shard; the loss (a sum over samples) and every gradient are
    summed over the ranks.  Each conv layer's weight gradient goes through
    fftconv_b200_grad_weight_sharded when `comm` (a sharded.NcclComm) is
    given -- chunked c2r, all-reduces on a side stream that overlap the rest
    of the backward pass, one wait at the end -- otherwise through
    torch.distributed all_reduce; the fc gradients through torch."""
    import torch
    import torch.distributed as dist

    sh = spec.shape()
    if len(params.conv) != sh.conv_count:
        raise ConfigError("run_iteration: wrong number of weight tensors")
    if batch.shape[1] != spec.input_maps:
        raise ConfigError(f"run_iteration: batch has {batch.shape[1]} maps, network wants {spec.input_maps}")
    dev = torch.device("cuda", device)
    x = batch if isinstance(batch, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(batch))
    x = x.to(dev).contiguous()
    S = x.shape[0]
    if ws is None:
        ws = ConvWorkspace(spec.conv_configs(S), device=device)
    multi = dist.is_available() and dist.is_initialized() and (dist.get_world_size(group) > 1 or comm is not None)
    sharded = None
    if multi and comm is not None:
        from .sharded import ShardedConv

        sharded = ShardedConv(ws, group=group, comm=comm, chunks=chunks)
    raw_ws = ws
    ws = _CountingWorkspace(ws)
    _LAUNCHES[0] = 0
    w_dev = [torch.from_numpy(np.ascontiguousarray(w)).to(dev) for w in params.conv]
    if sh.has_fc:
        fc_w = torch.from_numpy(np.ascontiguousarray(params.fc_weights)).to(dev)
        fc_b = torch.from_numpy(np.ascontiguousarray(params.fc_bias)).to(dev)
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False  # the fc layer stays fp32 like the reference

    events = {"update_output_ms": [], "update_grad_input_ms": [], "acc_grad_ms": []}

    def timed(bucket, fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn()
        e1.record()
        events[bucket].append((e0, e1))
        return r

    try:
        conv_rec, relu_rec, pool_rec = [], [], []
        # the backward's fit_to crops folded into grad_input's K4 crop
        # (fftconv_b200_grad_input_fit: the same values, fewer written).  The
        # forward pad stays explicit: folding it too (forward_fit on the
        # unpadded planes) is exact in real arithmetic, but K1's zero-pruned
        # transforms round differently, and outputs whose receptive field is
        # all padding (exactly 0) then come out as different +-1e-7 noise --
        # relu / max-pool decisions on that noise flip and the gradients move
        # by ~1e-4 relative (measured on reference-net-small).
        fold_fit = os.environ.get("FFTCONV_B200_FOLD_FIT", "1") != "0"
        state = {"cur": x, "fc_in": None, "scores": None}

        def forward_all():
            ci = 0
            fused = False  # the last conv already applied this relu (fftconv_b200_forward_relu)
            for si, st in enumerate(spec.stages):
                cur = state["cur"]
                if st.kind == StageKind.conv:
                    fused = si + 1 < len(spec.stages) and spec.stages[si + 1].kind == StageKind.relu
                    fin = fit_to(cur, st.conv.image)
                    # a padded input's gradient is cropped back inside K4 (below)
                    conv_rec.append((fin, cur.shape[2], fold_fit and cur.shape[2] < st.conv.image))
                    state["cur"] = ws.forward(fin, w_dev[ci], relu=fused)
                    ci += 1
                elif st.kind == StageKind.relu:
                    # relu backward masks by x > 0, and relu(x) > 0 exactly where x > 0,
                    # so the fused output serves as the record
                    relu_rec.append(cur)
                    if not fused:
                        state["cur"] = relu_forward(cur)
                    fused = False
                elif st.kind == StageKind.pool:
                    rec = maxpool_forward(cur)
                    pool_rec.append(rec)
                    state["cur"] = rec[0]
                elif st.kind == StageKind.fc:
                    state["fc_in"] = cur.reshape(S, -1)
                    state["scores"] = torch.addmm(fc_b, state["fc_in"], fc_w.t())
            final = state["scores"] if sh.has_fc else state["cur"]
            return final.double().sum()

        loss_t = timed("update_output_ms", forward_all)

        conv_grads = [None] * sh.conv_count
        fc_gw = fc_gb = None
        grad_input_calls = 0
        if sh.has_fc:
            gscores = torch.ones((S, sh.fc_outputs), dtype=torch.float32, device=dev)

            def fc_params():
                return gscores.t().mm(state["fc_in"]), gscores.sum(0)

            fc_gw, fc_gb = timed("acc_grad_ms", fc_params)
            grad = timed("update_grad_input_ms",
                         lambda: gscores.mm(fc_w).reshape(S, sh.final_maps, sh.final_size, sh.final_size))
        else:
            grad = torch.ones((S, sh.final_maps, sh.final_size, sh.final_size), dtype=torch.float32, device=dev)

        ci = sh.conv_count
        ri, pi = len(relu_rec), len(pool_rec)
        rstages = list(reversed(spec.stages))
        fuse_pool_relu = os.environ.get("FFTCONV_B200_POOL_RELU_FUSE", "1") != "0"
        relu_done = False  # the pool backward already applied this relu's mask
        for si, st in enumerate(rstages):
            if st.kind == StageKind.conv:
                ci -= 1
                fin, pre, crop_in_k4 = conv_rec[ci]
                g = grad
                if sharded is not None:  # all-reduce overlaps the remaining backward layers
                    def acc(g=g, fin=fin):
                        r = sharded.grad_weight_async(g, fin)
                        _launched(raw_ws.last_launch_count())
                        return r
                    conv_grads[ci] = timed("acc_grad_ms", acc)
                else:
                    conv_grads[ci] = timed("acc_grad_ms", lambda g=g, fin=fin: ws.grad_weight(g, fin))
                if ci > 0:
                    if crop_in_k4:  # fftconv_b200_grad_input_fit: fit_to's crop inside K4
                        grad = timed("update_grad_input_ms",
                                     lambda g=g, c=ci, pre=pre: ws.grad_input(g, w_dev[c], size=pre))
                    else:
                        grad = timed("update_grad_input_ms",
                                     lambda g=g, c=ci, pre=pre: fit_to(ws.grad_input(g, w_dev[c]), pre))
                    grad_input_calls += 1
                else:
                    break
            elif st.kind == StageKind.relu:
                ri -= 1
                if relu_done:
                    relu_done = False
                    continue
                grad = timed("update_grad_input_ms", lambda g=grad, r=relu_rec[ri]: relu_backward(g, r))
            elif st.kind == StageKind.pool:
                pi -= 1
                if fuse_pool_relu and si + 1 < len(rstages) and rstages[si + 1].kind == StageKind.relu:
                    # relu -> pool in the forward order: the relu's backward fused in
                    grad = timed("update_grad_input_ms",
                                 lambda g=grad, r=pool_rec[pi]: maxpool_relu_backward(g, r))
                    relu_done = True
                else:
                    grad = timed("update_grad_input_ms", lambda g=grad, r=pool_rec[pi]: maxpool_backward(g, r))

        if multi:
            def reduce_all():
                if sharded is not None:
                    sharded.wait()
                else:
                    for g in conv_grads:
                        dist.all_reduce(g, group=group)
                if sh.has_fc:
                    dist.all_reduce(fc_gw, group=group)
                    dist.all_reduce(fc_gb, group=group)
                lt = loss_t.reshape(1).clone()
                dist.all_reduce(lt, group=group)
                return lt
            loss_t = timed("acc_grad_ms", reduce_all)
        torch.cuda.synchronize(dev)
        times = StageTimes(**{k: sum(a.elapsed_time(b) for a, b in v) for k, v in events.items()})
        checksum = sum(float(g.double().sum()) for g in conv_grads)
        if sh.has_fc:
            checksum += float(fc_gw.double().sum()) + float(fc_gb.double().sum())
        return IterationResult(times, float(loss_t), conv_grads, fc_gw, fc_gb, grad_input_calls, checksum,
                               _LAUNCHES[0])
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
