"""World-size-2 test of the minibatch-sharded operators on CPU (gloo).

The per-rank workspace here is a test double driven by the CPU oracle (the
GPU box runs the same ShardedConv over the B200 workspace with NCCL); what is
checked is the sharding contract itself: y / gx concatenate over ranks and
gw, all-reduced, equals the full-batch gradient (conv_direct_test.cpp:186-212).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1312_5851_b200.sharded import ShardedConv, shard_range

CFG = (5, 12, 3, 4, 5)  # k, n, f, f', S (S odd: uneven shards)


class OracleWorkspace:
    def forward(self, x, w):
        return oracle.forward_fft(x, w)

    def grad_input(self, gy, w):
        return oracle.grad_input_fft(gy, w)

    def grad_weight(self, gy, x):
        return oracle.grad_weight_fft(gy, x)


def _inputs():
    k, n, f, fo, S = CFG
    no = n - k + 1
    x = oracle.fill_uniform((S, f, n, n), 7, 1, dtype=np.float64)
    w = oracle.fill_uniform((fo, f, k, k), 7, 2, dtype=np.float64)
    gy = oracle.fill_uniform((S, fo, no, no), 7, 3, dtype=np.float64)
    return x, w, gy


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, gy = _inputs()
        b0, b1 = shard_range(x.shape[0], world, rank)
        sc = ShardedConv(OracleWorkspace())
        y = sc.forward(x[b0:b1], w)
        gx = sc.grad_input(gy[b0:b1], w)
        gw = sc.grad_weight(gy[b0:b1], x[b0:b1])
        q.put((rank, b0, b1, y, gx, gw.numpy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(180)
def test_sharded_ops_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=150) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, w, gy = _inputs()
    y_full = oracle.forward_fft(x, w)
    gx_full = oracle.grad_input_fft(gy, w)
    gw_full = oracle.grad_weight_fft(gy, x)
    y = np.concatenate([r[3] for r in res])
    gx = np.concatenate([r[4] for r in res])
    assert [r[1:3] for r in res] == [(0, 3), (3, 5)]
    assert oracle.max_rel_error(y, y_full) < 1e-13
    assert oracle.max_rel_error(gx, gx_full) < 1e-13
    for r in res:  # every rank holds the all-reduced gradient
        assert oracle.max_rel_error(r[5], gw_full) < 1e-12


class OracleWorkspace32(OracleWorkspace):
    """fp32 results like the B200 workspace (an empty shard contributes fp32 zeros)."""

    def grad_weight(self, gy, x):
        return oracle.grad_weight_fft(gy, x).astype(np.float32)


def _worker_empty(rank, world, port, q):
    """S = 1 over two ranks: rank 1's shard is empty."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, w, gy = _inputs()
        x, gy = x[:1], gy[:1]
        b0, b1 = shard_range(1, world, rank)
        sc = ShardedConv(OracleWorkspace32())
        y = sc.forward(x[b0:b1], w)
        gx = sc.grad_input(gy[b0:b1], w)
        gw = sc.grad_weight(gy[b0:b1], x[b0:b1])
        q.put((rank, b0, b1, y.shape, gx.shape, gw.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_sharded_empty_shard_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_empty, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=150) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, w, gy = _inputs()
    gw_full = oracle.grad_weight_fft(gy[:1], x[:1])
    k, n, f, fo, S = CFG
    no = n - k + 1
    assert [r[1:3] for r in res] == [(0, 1), (1, 1)]
    assert res[0][3] == (1, fo, no, no) and res[1][3] == (0, fo, no, no)
    assert res[1][4] == (0, f, n, n)
    for r in res:
        assert oracle.max_rel_error(r[5], gw_full) < 1e-6
