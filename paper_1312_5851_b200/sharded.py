"""Minibatch (S) sharding of the three operators across ranks.

Batch decomposability (conv_direct_test.cpp:186-212): y and gx
of a minibatch are the concatenation of the per-slice results, gw is the sum
of the per-slice gradients.  So with x/gy sharded over ranks and w
replicated, fprop and bprop need no communication and accGrad needs one
all-reduce of the *spatial* f'*f*k*k gradient (1.8 MB at the paper point,
31.7 MB for the wide layer) -- reducing after the local c2r+crop moves 22-35x
fewer bytes than reducing spectra.

Two collective paths:

* ``NcclComm`` + the C ABI (``fftconv_b200_grad_weight_sharded``, the
  product path on GPUs): accGrad's final c2r runs in f'-row chunks and each
  chunk's gw rows are all-reduced over NCCL / NVLink on a side stream while
  the next chunk transforms.  The communicator is created by the library
  from a unique id that rank 0 broadcasts over the torch.distributed group.
* torch.distributed ``all_reduce`` of the finished gw (any backend; gloo for
  the CPU tests and numpy operands).
"""
from __future__ import annotations

import ctypes as C

from . import _native
from .errors import raise_for_status


def shard_range(S: int, world: int, rank: int):
    """Contiguous slice [b0, b1) of the minibatch owned by `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(S, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def _empty_like_slice(t, shape):
    import numpy as np

    if type(t).__module__.startswith("torch"):
        import torch

        return torch.empty(shape, dtype=torch.float32, device=t.device)
    return np.empty(shape, dtype=np.float32)


class NcclComm:
    """An NCCL communicator owned by libfftconv_b200 (include/fftconv_b200.h,
    fftconv_b200_nccl_comm_create): rank 0 draws the unique id, the
    torch.distributed group broadcasts it, every rank joins on `device`."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist

        L = _native.lib()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            raise_for_status(L.fftconv_b200_nccl_get_unique_id(uid), _native.last_error(None))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        h = C.c_void_p()
        raise_for_status(L.fftconv_b200_nccl_comm_create(uid, self.world, self.rank, int(device), C.byref(h)),
                         _native.last_error(None))
        self.handle = h

    @classmethod
    def single(cls, device: int):
        """A one-rank communicator (no process group): the sharded entry point
        on one GPU, as the tests use it."""
        self = cls.__new__(cls)
        L = _native.lib()
        uid = (C.c_uint8 * 128)()
        raise_for_status(L.fftconv_b200_nccl_get_unique_id(uid), _native.last_error(None))
        h = C.c_void_p()
        raise_for_status(L.fftconv_b200_nccl_comm_create(uid, 1, 0, int(device), C.byref(h)),
                         _native.last_error(None))
        self.handle, self.rank, self.world = h, 0, 1
        return self

    def close(self):
        if getattr(self, "handle", None):
            _native.lib().fftconv_b200_nccl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedConv:
    """fprop / bprop / accGrad of one layer with this rank's minibatch slice.

    `ws` is any object with the ConvWorkspace operator interface (the B200
    workspace on GPUs); `group` a torch.distributed process group (None =
    default).  With `comm` (an NcclComm) and CUDA operands, accGrad goes
    through the library's chunked, overlapped all-reduce; otherwise through
    torch.distributed.
    """

    def __init__(self, ws, group=None, comm: NcclComm | None = None, chunks: int = 4):
        self.ws = ws
        self.group = group
        self.comm = comm
        self.chunks = int(chunks)

    def forward(self, x_local, w):
        if int(x_local.shape[0]) == 0:  # empty shard: an empty slice of y
            k = int(w.shape[2])
            return _empty_like_slice(x_local, (0, int(w.shape[0]), int(x_local.shape[2]) - k + 1,
                                               int(x_local.shape[3]) - k + 1))
        return self.ws.forward(x_local, w)

    def grad_input(self, gy_local, w):
        if int(gy_local.shape[0]) == 0:
            k = int(w.shape[2])
            return _empty_like_slice(gy_local, (0, int(w.shape[1]), int(gy_local.shape[2]) + k - 1,
                                                int(gy_local.shape[3]) + k - 1))
        return self.ws.grad_input(gy_local, w)

    def grad_weight(self, gy_local, x_local):
        import torch
        import torch.distributed as dist

        if self.comm is not None and isinstance(gy_local, torch.Tensor) and gy_local.is_cuda:
            return self._grad_weight_nccl(gy_local, x_local)
        if self.comm is not None and not isinstance(gy_local, torch.Tensor):
            return self._grad_weight_nccl_host(gy_local, x_local)
        multi = dist.is_initialized() and dist.get_world_size(self.group) > 1
        if int(gy_local.shape[0]) == 0 and int(x_local.shape[0]) == 0:
            # empty shard (world > S): contribute zeros so the other ranks'
            # all-reduce still completes (the local operator would raise)
            fo, f = int(gy_local.shape[1]), int(x_local.shape[1])
            k = int(x_local.shape[2]) - int(gy_local.shape[2]) + 1
            if isinstance(gy_local, torch.Tensor):
                gw = torch.zeros((fo, f, k, k), dtype=torch.float32, device=gy_local.device)
            else:
                gw = torch.zeros((fo, f, k, k), dtype=torch.float32)
        else:
            gw = self.ws.grad_weight(gy_local, x_local)
        if not isinstance(gw, torch.Tensor):
            gw = torch.from_numpy(gw)
        if multi:
            if dist.get_backend(self.group) == "nccl" and not gw.is_cuda:
                # host-path result (numpy operands): NCCL reduces device buffers only
                gw = gw.to(torch.device("cuda", torch.cuda.current_device()))
            dist.all_reduce(gw, op=dist.ReduceOp.SUM, group=self.group)
        return gw

    def grad_weight_async(self, gy_local, x_local):
        """accGrad whose all-reduce keeps running behind the caller's next
        work (FFTCONV_B200_SHARDED_ASYNC); call wait() before reading gw."""
        return self._grad_weight_nccl(gy_local, x_local, flags=1)

    def wait(self):
        """The current stream waits for every all-reduce issued so far."""
        import torch

        code = _native.lib().fftconv_b200_comm_wait(self.ws._h, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        raise_for_status(code, _native.last_error(self.ws._h))

    def _grad_weight_nccl(self, gy, x, flags=0):
        """conv_fft.hpp:154-206 over the whole sharded minibatch, via
        fftconv_b200_grad_weight_sharded (include/fftconv_b200.h)."""
        import torch

        ws = self.ws
        Sg, fo, gr, gc = (int(v) for v in gy.shape)
        Sx, f, xr, xc = (int(v) for v in x.shape)
        k = xr - gr + 1 if gr <= xr else 1
        gw = torch.empty((fo, f, k, k), dtype=torch.float32, device=gy.device)
        code = _native.lib().fftconv_b200_grad_weight_sharded(
            ws._h, ws._dev_ptr(gy), Sg, fo, gr, gc, ws._dev_ptr(x), Sx, f, xr, xc,
            ws._dev_ptr(gw), self.comm.handle, self.chunks, int(flags),
            C.c_void_p(torch.cuda.current_stream(gy.device).cuda_stream))
        raise_for_status(code, _native.last_error(ws._h))
        return gw

    def _grad_weight_nccl_host(self, gy, x):
        """Host-buffer form (fftconv_b200_grad_weight_sharded_host): numpy
        shards in, the full-batch gradient (numpy) out."""
        import numpy as np

        gy = np.ascontiguousarray(gy, dtype=np.float32)
        x = np.ascontiguousarray(x, dtype=np.float32)
        Sg, fo, gr, gc = gy.shape
        Sx, f, xr, xc = x.shape
        k = xr - gr + 1 if gr <= xr else 1
        gw = np.zeros((fo, f, k, k), dtype=np.float32)
        code = _native.lib().fftconv_b200_grad_weight_sharded_host(
            self.ws._h, gy.ctypes.data_as(C.c_void_p), Sg, fo, gr, gc, x.ctypes.data_as(C.c_void_p), Sx, f, xr,
            xc, gw.ctypes.data_as(C.c_void_p), self.comm.handle, 1)
        raise_for_status(code, _native.last_error(self.ws._h))
        return gw

    def comm_ms(self):
        """(collective span, exposed) ms of the last timed sharded accGrad."""
        out = (C.c_float * 2)()
        code = _native.lib().fftconv_b200_comm_ms(self.ws._h, out)
        raise_for_status(code, _native.last_error(self.ws._h))
        return float(out[0]), float(out[1])
