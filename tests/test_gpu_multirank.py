"""The N>1 bench path (minibatch sharding + all-reduce of gw) end to end on
whatever GPUs the box has: two ranks via torchrun, gloo so they may share a
single GPU.  NCCL itself is exercised by the driver's multi-GPU runs."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "small", "--dist-backend", "gloo"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    # strong scaling by default (BASELINE configs[3]): the S=8 minibatch split 4 + 4
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    assert line["run"]["S_per_gpu"] == 4 and line["run"]["global_batch"] == 8
    assert line["config"]["S"] == 8
    mg = line["multi_gpu"]
    assert mg["grad_weight_sharded_ms"] > 0 and mg["max_over_ranks"]
    r = subprocess.run(cmd[:6] + [f"--master-port={_port()}"] + cmd[7:] + ["--weak"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert line["scaling"] == "weak" and line["run"]["S_per_gpu"] == 8 and line["run"]["global_batch"] == 16


def test_sharded_grad_weight_matches_full_batch(dev):
    """Two 'ranks' on one GPU in one process: per-slice gw summed == full gw."""
    import numpy as np
    import torch

    import oracle
    from paper_1312_5851_b200 import ConvWorkspace, LayerConfig
    from paper_1312_5851_b200.sharded import shard_range

    k, n, f, fo, S = 7, 32, 24, 20, 10
    x = oracle.fill_uniform((S, f, n, n), 3, 1)
    gy = oracle.fill_uniform((S, fo, n - k + 1, n - k + 1), 3, 3)
    full = ConvWorkspace([LayerConfig(k, n, f, fo, S)]).grad_weight(torch.from_numpy(gy).to(dev),
                                                                   torch.from_numpy(x).to(dev))
    parts = []
    for r in range(3):
        b0, b1 = shard_range(S, 3, r)
        ws = ConvWorkspace([LayerConfig(k, n, f, fo, b1 - b0)])
        parts.append(ws.grad_weight(torch.from_numpy(gy[b0:b1]).to(dev), torch.from_numpy(x[b0:b1]).to(dev)))
    tot = sum(parts).cpu().numpy()
    assert oracle.max_rel_error(tot, full.cpu().numpy()) < 1e-5
    del np


def test_stack_two_ranks_gloo_matches_one_rank():
    """The data-parallel training step (BASELINE configs[4] on N GPUs): two
    ranks each run half the minibatch of the reference-net-small stack; the
    summed loss and gradient checksum match the one-rank iteration."""
    base = [os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "3", "--config",
            "stack:reference-net-small"]
    r1 = subprocess.run([sys.executable] + base, capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    one = json.loads([l for l in r1.stdout.splitlines() if l.startswith("{")][0])
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}"] + base + ["--gpus", "2", "--dist-backend", "gloo"]
    r2 = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r2.returncode == 0, r2.stderr[-3000:]
    lines = [l for l in r2.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    two = json.loads(lines[0])
    assert two["n_gpus"] == 2 and two["run"]["S_per_gpu"] == 4 and two["value"] > 0
    assert abs(two["loss"] - one["loss"]) <= 1e-5 * abs(one["loss"])
    assert abs(two["grad_checksum"] - one["grad_checksum"]) <= 1e-4 * abs(one["grad_checksum"])
