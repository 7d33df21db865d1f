"""The minibatch-sharded accGrad entry point (include/fftconv_b200.h,
fftconv_b200_grad_weight_sharded) on a one-rank NCCL communicator created by
the library: chunked c2r + per-chunk all-reduce must reproduce grad_weight
bit for bit (a one-rank all-reduce is a copy; the chunks run the same
arithmetic per plane group), at every FFT-size family (m = 16 / 32 TMA K4 on
group-major products, m = 64 on bin-major ones, m = 128 two-pass), for
ragged f' and empty shards.  Multi-rank NCCL needs one GPU per rank (the
driver's multi-GPU runs); the orchestration is covered with gloo in
test_sharding_gloo.py / test_gpu_multirank.py."""
import numpy as np
import pytest

import oracle
from paper_1312_5851_b200 import ConvWorkspace, LayerConfig
from paper_1312_5851_b200.sharded import NcclComm, ShardedConv

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    c = NcclComm.single(0)
    yield c
    c.close()


def _inputs(cfg, seed):
    S, f, fo, n, k = cfg.batch, cfg.in_maps, cfg.out_maps, cfg.image, cfg.kernel
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), seed, oracle.ROLE_INPUT)
    gy = oracle.fill_uniform((S, fo, no, no), seed, oracle.ROLE_GRAD_OUTPUT)
    return x, gy


@pytest.mark.parametrize("cfg", [(7, 32, 96, 96, 128), (5, 16, 24, 40, 12), (11, 64, 32, 70, 6),
                                 (9, 100, 3, 20, 2), (3, 8, 5, 33, 4)])
@pytest.mark.parametrize("chunks", [1, 3, 4, 16])
def test_sharded_equals_local_grad_weight(dev, comm, cfg, chunks):
    import torch

    cfg = LayerConfig(*cfg)
    x, gy = _inputs(cfg, 61)
    ws = ConvWorkspace([cfg])
    xd, gyd = torch.from_numpy(x).to(dev), torch.from_numpy(gy).to(dev)
    ref = ws.grad_weight(gyd, xd)
    got = ShardedConv(ws, comm=comm, chunks=chunks).grad_weight(gyd, xd)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    if chunks == 4:
        x64, gy64 = x.astype(np.float64), gy.astype(np.float64)
        assert oracle.rel_l2_error(got.cpu().numpy(), oracle.grad_weight_fft(gy64, x64)) <= 1e-4


def test_sharded_empty_shard_contributes_zeros(dev, comm):
    import torch

    cfg = LayerConfig(5, 16, 4, 6, 2)
    ws = ConvWorkspace([cfg])
    x = torch.zeros((0, 4, 16, 16), device=dev)
    gy = torch.zeros((0, 6, 12, 12), device=dev)
    gw = ShardedConv(ws, comm=comm).grad_weight(gy, x)
    torch.cuda.synchronize()
    assert gw.shape == (6, 4, 5, 5) and float(gw.abs().max()) == 0.0


def test_sharded_comm_timing(dev, comm):
    import torch

    cfg = LayerConfig(7, 32, 96, 96, 128)
    x, gy = _inputs(cfg, 62)
    ws = ConvWorkspace([cfg])
    sc = ShardedConv(ws, comm=comm, chunks=4)
    xd, gyd = torch.from_numpy(x).to(dev), torch.from_numpy(gy).to(dev)
    ws.set_stage_timing(True)
    sc.grad_weight(gyd, xd)
    span, exposed = sc.comm_ms()
    ws.set_stage_timing(False)
    assert span > 0 and 0 <= exposed
    assert ws.last_launch_count() >= 2 + 4  # K1, K3 and four K4 chunks


def test_run_iteration_through_sharded_accgrad(dev, comm):
    """The data-parallel training step's conv gradients via the async sharded
    entry point (all-reduces behind the backward pass, one wait at the end)
    on a one-rank group equal the plain iteration's."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1312_5851_b200 import layers

    spec = layers.preset_network("reference-net-small")
    params = layers.init_params(spec, 5)
    batch = layers.make_batch(spec, spec.default_batch, 5)
    plain = layers.run_iteration(spec, params, batch)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        dp = layers.run_iteration(spec, params, batch, comm=comm)
    finally:
        dist.destroy_process_group()
    torch.cuda.synchronize()
    assert dp.loss == plain.loss
    for a, b in zip(dp.conv_weight_grads, plain.conv_weight_grads):
        assert torch.equal(a, b)
    assert torch.equal(dp.fc_weight_grad, plain.fc_weight_grad)


def test_sharded_host_buffers(comm):
    """fftconv_b200_grad_weight_sharded_host (the drop-in's Tensor4 storage):
    numpy shards in, the all-reduced gradient out; an empty shard gives zeros."""
    cfg = LayerConfig(7, 32, 24, 20, 10)
    x, gy = _inputs(cfg, 63)
    ws = ConvWorkspace([cfg])
    ref = ws.grad_weight(gy, x)  # host path
    got = ShardedConv(ws, comm=comm).grad_weight(gy, x)
    assert isinstance(got, np.ndarray) and np.array_equal(got, ref)
    ez = ShardedConv(ws, comm=comm).grad_weight(np.zeros((0, 20, 26, 26), np.float32),
                                                 np.zeros((0, 24, 32, 32), np.float32))
    assert ez.shape == (20, 24, 7, 7) and not ez.any()
