"""Per-iteration stage times of a layer-stack preset (5 iterations), to spot
outliers: python tools/dev/stack_times.py alexnet-128"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1312_5851_b200 import ConvWorkspace, layers  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "alexnet-128"
spec = layers.preset_network(name)
S = spec.default_batch
params = layers.init_params(spec, 1234)
batch = torch.from_numpy(layers.make_batch(spec, S, 1234)).cuda()
ws = ConvWorkspace(spec.conv_configs(S), device=0)
for i in range(int(os.environ.get('ITERS', 6))):
    t0 = time.perf_counter()
    r = layers.run_iteration(spec, params, batch, ws=ws)
    t1 = time.perf_counter()
    ms = torch.cuda.memory_stats()
    print(i, round((t1 - t0) * 1e3, 2), "ms wall", r.times, torch.cuda.memory_allocated() >> 20, "MiB",
          "retries", ms.get("num_alloc_retries"), "device allocs", ms.get("num_device_alloc"),
          "frees", ms.get("num_device_free"), flush=True)
