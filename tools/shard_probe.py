"""Per-rank step time of the view-sharded path, emulated on one GPU: the c4 step over V/N of its views
(what one of N ranks computes), with the static cache, as a CUDA-graph replay -- the bench's N > 1 form
minus the all-reduce of the packed active rows (one NCCL collective of (4 + A x 60) floats per step,
captured in the same graph; it cannot run across ranks on this one-GPU box).  Prints ms per step."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
sc = synth.make_scene(cfg)
V = len(sc.cameras)
out = {}
for N in (1, 2, 4, 8):
    views = list(range(V // N))
    cams = [sc.cameras[v] for v in views]
    params = GaussianParams.from_scene(sc, device="cuda:0")
    lim = bench.limits_for(cfg, sc.n, len(cams), sc.width, sc.height, False)
    lim.max_active = 32768
    opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True)
    opt.spatial_order()
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets[views])).cuda()
    opt.step(cams, tg, n_views_total=V)
    g = GraphStep(opt, cams, tg, n_views_total=V)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    out[N] = round(ms, 4)
    print(f"N={N}: {len(cams)} views/rank: graph {ms:.3f} ms/step (rank work, no all-reduce)", flush=True)
    opt.close()
    del params, opt, g
    torch.cuda.empty_cache()
print(json.dumps({"config": cfg, "per_rank_ms": out, "projected_speedup_8": round(out[1] / out[8], 2)}))
