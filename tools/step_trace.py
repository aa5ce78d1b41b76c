"""Per-step device times of consecutive CUDA-graph replays of the c4 (argv[1]) step, and the static cache's
build count over them: how the step time evolves after the cache build (warm-up, rebuilds)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 120
sc = synth.make_scene(cfg)
u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for(cfg, sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
opt.spatial_order()
td = torch.from_numpy(u8).cuda()
g = GraphStep(opt, sc.cameras, td)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
ev[0].record()
for k in range(n):
    g.replay()
    ev[k + 1].record()
torch.cuda.synchronize()
ms = [round(ev[k].elapsed_time(ev[k + 1]), 3) for k in range(n)]
if "--clocks" in sys.argv:   # SM clock right after the loop, then a second loop after the GPU idled 1 s
    import subprocess
    import time
    q = ["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw", "--format=csv,noheader"]
    print("clock after loop", subprocess.run(q, capture_output=True, text=True).stdout.strip())
    time.sleep(1.0)
    print("clock idle", subprocess.run(q, capture_output=True, text=True).stdout.strip())
    ev[0].record()
    for k in range(n):
        g.replay()
        ev[k + 1].record()
    torch.cuda.synchronize()
    ms2 = [round(ev[k].elapsed_time(ev[k + 1]), 3) for k in range(n)]
    print("second loop", [round(float(np.mean(ms2[i:i + 10])), 3) for i in range(0, n, 10)])
st = opt.stats()
print(json.dumps({"config": cfg, "step_ms": ms, "builds": st["cache_builds"], "mask_builds": st["cache_mask_builds"],
                  "dilation": st["cache_dilation"]}))
