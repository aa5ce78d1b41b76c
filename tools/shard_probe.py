"""Per-rank step time of the view-sharded path, emulated on one GPU: the step over V/N of c4's views
(what one of N ranks computes; the all-reduce of the active rows is not included).  Eager steps, as
bench.py runs at N > 1, and graph replay for comparison."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import synth
import bench
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer

sc = synth.make_scene("c4")
V = len(sc.cameras)
for N in (1, 2, 4, 8):
    views = list(range(V // N))
    cams = [sc.cameras[v] for v in views]
    params = GaussianParams.from_scene(sc, device="cuda:0")
    lim = bench.limits_for("c4", sc.n, len(cams), sc.width, sc.height, False)
    opt = LocalOptimizer(params, sc.regions, limits=lim)
    opt.spatial_order()
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets[views])).cuda()
    res = {}
    for mode in ("eager", "graph"):
        if mode == "graph":
            g = GraphStep(opt, cams, tg, n_views_total=V)
            step = g.replay
        else:
            step = lambda: opt.step(cams, tg, n_views_total=V)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            step()
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 20
    print(f"N={N}: {len(cams)} views/rank: eager {res['eager']:.3f} ms, graph {res['graph']:.3f} ms")
    opt.close()
    del params
    torch.cuda.empty_cache()
