import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import synth, bench
from paper_2506_21117_b200 import GaussianParams, LocalOptimizer
sc = synth.make_scene("c4")
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c4", sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim)
opt.spatial_order()
tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).pin_memory()
for _ in range(3):
    opt.step(sc.cameras, tg)
torch.cuda.synchronize()
opt.profile(True); opt.profile_read()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    opt.step(sc.cameras, tg)
e1.record(); torch.cuda.synchronize()
pr = opt.profile_read()
print("ms/step", e0.elapsed_time(e1) / 10)
print({k: round(v["ms"] / max(v["calls"], 1), 4) for k, v in pr.items() if v["calls"]})
