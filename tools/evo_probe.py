import sys, json
import numpy as np, torch
sys.path.insert(0, '.')
import bench, synth
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer
sc = synth.make_scene("c4")
u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c4", sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
opt.spatial_order()
td = torch.from_numpy(u8).cuda()
rows = []
for k in range(45):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    opt.step(sc.cameras, td)
    e1.record()
    torch.cuda.synchronize()
    st = opt.stats()
    rows.append((k, round(e0.elapsed_time(e1), 3), st["n_active"], st["n_records"], st["n_pairs"], st["n_items"], st["n_fwd_evals"], st["n_fwd_exec"], st["n_bwd_evals"], st["cache_mode"], st["max_list"]))
for r in rows: print(r)
