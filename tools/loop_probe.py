"""Per-step device time of BASELINE config 5's loop (bench.py --loop) with the static cache's mode of
each step: where the loop's time goes (warm steps, rebuilds, refreshes after a prune, re-captures)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402


class A:
    config = sys.argv[1] if len(sys.argv) > 1 else "c5"
    targets = "u8"
    no_spatial_order = False


sc, u8 = bench.bench_scene(A)
V = len(sc.cameras)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for(A.config, sc.n, V, sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True, per_set="--per-set" in sys.argv)
opt.spatial_order()
opt.partition_static()
tg = torch.from_numpy(np.ascontiguousarray(u8)).cuda()
for _ in range(3):
    opt.step(sc.cameras, tg)
torch.cuda.synchronize()
rows = []
gs = None
for k in range(100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    pr = 0
    if k > 0 and k % 15 == 0:
        pr = opt.prune_outside()
        gs = None
    cap = gs is None
    if gs is None:
        gs = GraphStep(opt, sc.cameras, tg)
    gs.replay()
    e1.record()
    torch.cuda.synchronize()
    st = opt.stats()
    rows.append((k, round(e0.elapsed_time(e1), 3), st["cache_mode"], int(cap), pr))
ms = [r[1] for r in rows]
print(json.dumps({"total_ms": round(sum(ms), 2), "median": sorted(ms)[50],
                  "slow": sorted(rows, key=lambda r: -r[1])[:16]}))
