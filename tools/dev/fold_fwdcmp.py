import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1312_5851_b200 import ConvWorkspace, layers
spec = layers.preset_network("reference-net-small")
S = spec.default_batch
params = layers.init_params(spec, 1234)
x = torch.from_numpy(layers.make_batch(spec, S, 1234)).cuda()
ws = ConvWorkspace(spec.conv_configs(S), device=0)
w = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in params.conv]
cur_a = cur_b = x
ci = 0
for st in spec.stages:
    if st.kind == layers.StageKind.conv:
        n = st.conv.image
        ya = ws.forward(layers.fit_to(cur_a, n), w[ci], relu=True)
        yb = ws.forward(cur_b, w[ci], relu=True, image=n) if cur_b.shape[2] < n else ws.forward(layers.fit_to(cur_b, n), w[ci], relu=True)
        # same input to both to isolate the operator
        yc = ws.forward(cur_a, w[ci], relu=True, image=n) if cur_a.shape[2] < n else ya
        d = (ya - yc).abs().max().item()
        print("conv", ci, "in", tuple(cur_a.shape), "max|fit - fold| (same input)", d, "exact zero diffs", int(((ya == 0) != (yc == 0)).sum()))
        cur_a, cur_b = ya, yb
        ci += 1
    elif st.kind == layers.StageKind.pool:
        ra, rb = layers.maxpool_forward(cur_a), layers.maxpool_forward(cur_b)
        print("pool argmax differences", int((ra[1] != rb[1]).sum()), "of", ra[1].numel())
        cur_a, cur_b = ra[0], rb[0]
