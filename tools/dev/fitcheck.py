import sys; sys.path.insert(0, '.')
import numpy as np, torch
import oracle
from paper_1312_5851_b200 import ConvWorkspace, layers
spec = layers.preset_network("reference-net-small")
S = spec.default_batch
ws = ConvWorkspace(spec.conv_configs(S), device=0)
rng = np.random.default_rng(3)
dev = torch.device("cuda:0")
pre_sizes = {32: [22], 16: [13, 12]}
for cfg in spec.conv_configs(S):
    k, n, f, fo = cfg.kernel, cfg.image, cfg.in_maps, cfg.out_maps
    for pre in pre_sizes.get(n, []):
        x = torch.from_numpy(rng.standard_normal((S, f, pre, pre)).astype(np.float32)).to(dev)
        w = torch.from_numpy(rng.standard_normal((fo, f, k, k)).astype(np.float32)).to(dev)
        no = n - k + 1
        gy = torch.from_numpy(rng.standard_normal((S, fo, no, no)).astype(np.float32)).to(dev)
        xp = layers.fit_to(x, n)
        e = lambda a, b: oracle.rel_l2_error(a.cpu().numpy(), b.cpu().numpy())
        print(cfg, pre, "fwd", e(ws.forward(x, w, image=n), ws.forward(xp, w)),
              "gi", e(ws.grad_input(gy, w, size=pre), layers.fit_to(ws.grad_input(gy, w), pre)),
              "gw", e(ws.grad_weight(gy, x, image=n), ws.grad_weight(gy, xp)))
