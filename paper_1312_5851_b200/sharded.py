"""Minibatch (S) sharding of the three operators across ranks.

Batch decomposability (conv_direct_test.cpp:186-212): y and gx
of a minibatch are the concatenation of the per-slice results, gw is the sum
of the per-slice gradients.  So with x/gy sharded over ranks and w
replicated, fprop and bprop need no communication and accGrad needs one
all-reduce of the *spatial* f'*f*k*k gradient (1.8 MB at the paper point,
31.7 MB for the wide layer) -- reducing after the local c2r+crop moves 22-35x
fewer bytes than reducing spectra.

Works with any torch.distributed backend: NCCL over NVLink on the GPU box,
gloo for the CPU tests.
"""
from __future__ import annotations


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


class ShardedConv:
    """fprop / bprop / accGrad of one layer with this rank's minibatch slice.

    `ws` is any object with the ConvWorkspace operator interface (the B200
    workspace on GPUs); `group` a torch.distributed process group (None =
    default).
    """

    def __init__(self, ws, group=None):
        self.ws = ws
        self.group = group

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
