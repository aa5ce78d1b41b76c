"""Per-kernel-group breakdown of ONE rank's share of the c4 step at N GPUs (views V/N), static cache:
the graph-replay time per step and the eager per-group event times (what bounds multi-GPU scaling)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sc = synth.make_scene("c4")
V = len(sc.cameras)
views = list(range(V // N))
cams = [sc.cameras[v] for v in views]
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c4", sc.n, len(cams), sc.width, sc.height, False)
lim.max_active = 32768
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
opt.spatial_order()
tg = torch.from_numpy(np.ascontiguousarray(sc.targets[views])).cuda()
opt.step(cams, tg, n_views_total=V)
g = GraphStep(opt, cams, tg, n_views_total=V)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    g.replay()
e1.record()
torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1) / 50
opt.profile(True)
opt.profile_read()
for _ in range(20):
    opt.step(cams, tg, n_views_total=V)
torch.cuda.synchronize()
prof = opt.profile_read()
br = {k: round(v["ms"] / 20, 4) for k, v in prof.items() if v["calls"]}
print(json.dumps({"N": N, "views": len(cams), "graph_ms": round(graph_ms, 4), "eager_group_ms": br,
                  "eager_sum": round(sum(br.values()), 4)}))
