"""(ncu helper) capture the c4 warm step as a graph and replay it a few times; run under
`ncu --metrics gpu__time_duration.sum` to list the graph's kernel nodes in order."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
sc = synth.make_scene(cfg)
u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for(cfg, sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
opt.spatial_order()
td = torch.from_numpy(u8).cuda()
g = GraphStep(opt, sc.cameras, td)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
print("ok")
