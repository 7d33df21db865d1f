"""Pinned H2D / D2H throughput with 1 / 2 / 4 concurrent streams and with
both directions at once (is the host path's copy side link- or engine-bound?)."""
import time

import torch

dev = torch.device("cuda:0")
N = 256 << 20
h = [torch.empty(N // 4, dtype=torch.float32).pin_memory() for _ in range(4)]
d = [torch.empty(N // 4, dtype=torch.float32, device=dev) for _ in range(4)]
for x in h:
    x.fill_(1.0)


def run(nstreams, h2d=True, d2h=False, reps=3):
    ss = [torch.cuda.Stream() for _ in range(8)]
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k = 0
        if h2d:
            for i in range(4):
                with torch.cuda.stream(ss[i % nstreams]):
                    d[i].copy_(h[i], non_blocking=True)
        if d2h:
            for i in range(4):
                with torch.cuda.stream(ss[4 + i % nstreams]):
                    h[i].copy_(d[(i + 1) % 4], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    nbytes = 4 * N * (int(h2d) + int(d2h))
    return nbytes / best / 1e9


for ns in (1, 2, 4):
    print(f"H2D {ns} streams: {run(ns):.1f} GB/s   D2H: {run(ns, False, True):.1f} GB/s   "
          f"both: {run(ns, True, True):.1f} GB/s total")
