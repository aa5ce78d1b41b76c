"""Where the end-to-end step's time goes (c4, static cache, 8-bit targets): CUDA-graph replays over
device targets vs over pinned host targets, and the eager per-group times of the host-target step
(gather_targets runs on its own stream, overlapped)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402

sc = synth.make_scene("c4")
u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c4", sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
opt.spatial_order()
th = torch.from_numpy(u8).pin_memory()
td = th.cuda()
for name, tg in (("device", td), ("host", th)):
    g = GraphStep(opt, sc.cameras, tg)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(name, "graph ms/step", round(e0.elapsed_time(e1) / 20, 4), flush=True)
opt.profile(True)
opt.profile_read()
for _ in range(10):
    opt.step(sc.cameras, th)
torch.cuda.synchronize()
pr = opt.profile_read()
print({k: round(v["ms"] / max(v["calls"], 1), 4) for k, v in pr.items() if v["calls"]})
