import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import synth, bench
from paper_2506_21117_b200 import GaussianParams, LocalOptimizer
sc = synth.make_scene("c4")
V = len(sc.cameras)
views = list(range(4))
cams = [sc.cameras[v] for v in views]
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c4", sc.n, len(cams), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim)
opt.spatial_order()
tg = torch.from_numpy(np.ascontiguousarray(sc.targets[views])).cuda()
for _ in range(3):
    opt.step(cams, tg, n_views_total=V)
torch.cuda.synchronize()
opt.profile(True); opt.profile_read()
for _ in range(10):
    opt.step(cams, tg, n_views_total=V)
torch.cuda.synchronize()
pr = opt.profile_read()
print({k: round(v["ms"] / max(v["calls"], 1), 4) for k, v in pr.items() if v["calls"]})
print(opt.stats())
