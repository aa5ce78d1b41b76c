"""Host-side phases of BASELINE config 5's loop (bench.py --loop): wall time of every prune, every
GraphStep construction (eager warm-up step + capture + instantiate) and the replays, to find where the
loop's run-to-run variance comes from."""
import gc
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer  # noqa: E402


class A:
    config = "c5"
    targets = "u8"
    no_spatial_order = False


sc, u8 = bench.bench_scene(A)
params = GaussianParams.from_scene(sc, device="cuda:0")
lim = bench.limits_for("c5", sc.n, len(sc.cameras), sc.width, sc.height, False)
opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True, per_set="--per-set" in sys.argv)
opt.spatial_order()
opt.partition_static()
tg = torch.from_numpy(np.ascontiguousarray(u8)).cuda()
for _ in range(3):
    opt.step(sc.cameras, tg)
torch.cuda.synchronize()
if "--nogc" in sys.argv:
    gc.collect()
    gc.disable()
ph = {"prune": [], "graphstep": [], "replay": []}
gs = None
keep = []   # --keep: the re-captured steps stay alive until the end (no pool frees inside the loop)
t_all = time.perf_counter()
for k in range(100):
    if k > 0 and k % 15 == 0:
        t0 = time.perf_counter(); opt.prune_outside(); ph["prune"].append(time.perf_counter() - t0)
        if "--keep" in sys.argv:
            keep.append(gs)
        gs = None
    if gs is None:
        t0 = time.perf_counter(); gs = GraphStep(opt, sc.cameras, tg); ph["graphstep"].append(time.perf_counter() - t0)
        ph.setdefault("warmup", []).append(gs.host_ms["warmup"] / 1e3)
        ph.setdefault("capture", []).append(gs.host_ms["capture"] / 1e3)
        ph.setdefault("mode_after_warmup", []).append(int(opt.stats()["cache_mode"]))
    t0 = time.perf_counter(); gs.replay(); ph["replay"].append(time.perf_counter() - t0)
torch.cuda.synchronize()
total = time.perf_counter() - t_all
print(json.dumps({"total_s": round(total, 3), **{k: [round(x * 1e3, 1) for x in v] for k, v in ph.items() if k not in ("replay", "mode_after_warmup")},
                  "modes": ph.get("mode_after_warmup"),
                  "replay_ms_max": round(max(ph["replay"]) * 1e3, 2), "replay_ms_sum": round(sum(ph["replay"]) * 1e3, 1)}))
