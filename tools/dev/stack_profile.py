"""One training iteration of a layer-stack preset (for an ncu launch list):
python tools/dev/stack_profile.py alexnet-128"""
import os
import sys

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
for _ in range(2):
    layers.run_iteration(spec, params, batch, ws=ws)
torch.cuda.synchronize()
