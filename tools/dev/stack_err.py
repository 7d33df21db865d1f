"""Per-layer weight-gradient errors of run_iteration vs the reference's
run_iteration<float> and <double>: python tools/dev/stack_err.py [preset]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1312_5851_b200 import layers  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reference-net-small"
spec = layers.preset_network(name)
seed, S = 1234, spec.default_batch
params = layers.init_params(spec, seed)
batch = layers.make_batch(spec, S, seed)
res = layers.run_iteration(spec, params, batch)
f32, _ = oracle.ref_run_iteration(spec.records(), S, seed, engine=1)
f64, _ = oracle.ref_run_iteration(spec.records(), S, seed, engine=1, dtype=np.float64)
off = 0
for i, g in enumerate(res.conv_weight_grads):
    n = g.numel()
    a = g.cpu().numpy().reshape(-1).astype(np.float64)
    r32, r64 = f32[off:off + n], f64[off:off + n]
    e = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
    print(f"conv{i}: ours vs f32 {e(a, r32):.2e}  ours vs f64 {e(a, r64):.2e}  ref f32 vs f64 {e(r32, r64):.2e}")
    off += n
