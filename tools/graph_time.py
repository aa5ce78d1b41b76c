"""c4 (or argv[1]) warm graph-step time with device-resident 8-bit targets (A/B helper: run once per env)."""
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
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
res = []
for rep in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 20)
st = opt.stats()
print(cfg, "graph ms/step", [round(x, 4) for x in res], "min", round(min(res), 4), "loss", float(g.loss.item()),
      {k: st[k] for k in ("n_pairs", "n_records", "n_items") if k in st}, flush=True)
