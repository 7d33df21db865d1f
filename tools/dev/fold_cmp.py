"""run_iteration with the fit_to fold on and off: per-layer gradient
differences (debugging aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1312_5851_b200 import ConvWorkspace, layers  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "reference-net-small"
spec = layers.preset_network(name)
seed, S = 1234, spec.default_batch
params = layers.init_params(spec, seed)
batch = layers.make_batch(spec, S, seed)
out = {}
for v in ("0", "1"):
    os.environ["FFTCONV_B200_FOLD_FIT"] = v
    ws = ConvWorkspace(spec.conv_configs(S), device=0)
    out[v] = layers.run_iteration(spec, params, batch, ws=ws)
a, b = out["0"], out["1"]
print("loss", a.loss, b.loss)
for i, (x, y) in enumerate(zip(a.conv_weight_grads, b.conv_weight_grads)):
    x, y = x.cpu().numpy().astype(np.float64), y.cpu().numpy().astype(np.float64)
    print(i, x.shape, float(np.linalg.norm(x - y) / np.linalg.norm(x)))
x, y = a.fc_weight_grad.cpu().numpy(), b.fc_weight_grad.cpu().numpy()
print("fc", float(np.linalg.norm(x - y) / np.linalg.norm(x)))
