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
        return self.ws.forward(x_local, w)

    def grad_input(self, gy_local, w):
        return self.ws.grad_input(gy_local, w)

    def grad_weight(self, gy_local, x_local):
        import torch
        import torch.distributed as dist

        gw = self.ws.grad_weight(gy_local, x_local)
        if not isinstance(gw, torch.Tensor):
            gw = torch.from_numpy(gw)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(gw, op=dist.ReduceOp.SUM, group=self.group)
        return gw
