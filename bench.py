#!/usr/bin/env python
"""Benchmark of the CL-Splats local-optimisation step (fwd + bwd + masked Adam) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One step = one pass of the whole hot path (membership, tile mask, projection, binning,
masked compositing + fused L1, masked backward, [NCCL all-reduce of the active gradient
rows when N > 1], masked Adam) over all views of the config.  N > 1: run under
torch.distributed.run, one rank per GPU; the views are sharded over the ranks (weak in the
Gaussians, strong in the views: the total work per step is fixed).

Prints ONE JSON line (rank 0).  `value` = steps/s of the whole job, timed with CUDA events
on the launching stream over exactly K steps bracketed by barrier + synchronize, max over
ranks.  At N = 1 the step (fwd + bwd + masked Adam) is captured once as a CUDA graph and
replayed (`--eager` launches every kernel instead); the per-kernel breakdown then comes from
K eager steps run right after.  The roofline of the dominant kernel uses the library's own CUDA-event timing of
each kernel group over the same timed region.  `--impl reference` times the CPU oracle
(oracle/, fp64) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

# algorithmic FP32 FLOPs per (pixel, list entry) evaluation:
#   forward: LDL^T exponent 10, alpha 2, tests 2, transmittance 2, (composite 7 when composited)
#   backward walk: exponent 10, alpha 2, tests 2, T division 2, colour-behind 7
FWD_FLOPS_PER_EVAL = 19.5   # ~1.7 MFLOP per 256 px x 340 evaluations (incl. compositing)
BWD_FLOPS_PER_EVAL = 23.0
SM_COUNT, FP32_LANES = 148, 128


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init) can stall this process's driver calls for a long moment:
            # let it finish before the timed region (the loop's host work -- prunes, re-captures -- would
            # otherwise absorb it)
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.02)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in self.rows if num(r[0])]
        mx = [num(r[1]) for r in self.rows if num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[4 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def limits_for(cfg: str, n: int, n_views: int, W: int, H: int, all_tiles: bool):
    from paper_2506_21117_b200 import default_limits
    TX, TY = -(-W // 16), -(-H // 16)
    rec = n if (all_tiles or n <= 200_000) else n // 2   # records per view (capacity)
    pairs = min(TX * TY * 2048, 8_000_000 if not all_tiles else 24_000_000)
    pairs = min(pairs, (2**31 - 2) // max(n_views, 1))
    return default_limits(n, n_views, W, H, records_per_view=min(rec, (2**31 - 1) // max(n_views, 1)),
                          pairs_per_view=pairs, max_active=min(n, 400_000))


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2506_21117_b200.dist import allreduce_packed, shard_views
    sc, u8 = bench_scene(args)
    V = len(sc.cameras)
    my_views = shard_views(V, world, rank)
    cams = [sc.cameras[v] for v in my_views]
    W, H = sc.width, sc.height
    params = GaussianParams.from_scene(sc, device=f"cuda:{local}")
    lim = limits_for(args.config, sc.n, len(cams), W, H, args.all_tiles)
    cached = (args.static_cache == "on" or (args.static_cache == "auto" and sc.n >= 500_000)) and not args.all_tiles
    args.static_cache = cached
    if world > 1:
        # the all-reduce of a CUDA-graph step covers the gradient-row CAPACITY (max_active): size it from
        # |O^t| of the scene (one membership pass through the library) with headroom; a larger active set
        # is a reported overflow, never a silent truncation
        probe = LocalOptimizer(params, sc.regions, limits=lim)
        probe.forward(cams[:1], None)
        A = probe.active_count()
        probe.close()
        lim.max_active = max(1024, int(A * 1.25) + 256)
    opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=cached)
    if not args.no_spatial_order:
        opt.spatial_order()   # scene layout, once at load (not part of a step): Morton-ordered rows
    tg_np = u8[my_views] if u8 is not None else sc.targets[my_views]
    tg_host = torch.from_numpy(np.ascontiguousarray(tg_np)).pin_memory()
    tbytes = tg_host.element_size()
    tg = tg_host.to(f"cuda:{local}")
    stream = torch.cuda.current_stream()

    def step(targets=None):
        t = tg if targets is None else targets
        if world > 1:   # the step's only exchange: one NCCL all-reduce of the packed loss + active rows
            return opt.step(cams, t, n_views_total=V, allreduce=allreduce_packed)
        res = opt.forward(cams, t, n_views_total=V, all_tiles=args.all_tiles)
        grad = opt.backward()
        opt.adam(grad)
        return res.loss

    # cold step: an eager step that builds the static cache (after a first step that also allocated it:
    # a new content generation invalidates the cache, so the timed step rebuilds it from scratch)
    step()
    n_active0 = int(opt.stats()["n_active"])   # |O^t| of the initial scene (the workload's, as the reference arm's)
    params.touch()
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    step()
    c1.record(stream)
    torch.cuda.synchronize()
    cold_ms = c0.elapsed_time(c1)
    gstep = None
    graph_note = None
    if not args.eager and not args.all_tiles:
        from paper_2506_21117_b200 import GraphStep
        try:   # fwd + bwd (+ NCCL all-reduce at N > 1) + masked Adam captured once
            gstep = GraphStep(opt, cams, tg, n_views_total=V, allreduce=allreduce_packed if world > 1 else None)
            step_eager = step
            step = lambda targets=None: gstep.replay()
        except Exception as e:   # e.g. a NCCL build that cannot be captured: eager steps, said in step_mode
            torch.cuda.synchronize()
            gstep = None
            graph_note = f"graph capture failed ({type(e).__name__}: {str(e)[:120]}); eager steps"
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st0 = opt.stats()
    # ---------------- timed region (device) ----------------
    opt.profile(True)
    opt.profile_read()
    launches0 = opt.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            loss = step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_total = e0.elapsed_time(e1)
    launches = opt.launch_count() - launches0
    prof = opt.profile_read()
    if gstep is not None:
        # graph replays carry no per-kernel events and no host launches: the kernel breakdown and the
        # per-step kernel count come from K eager steps right after (same workload)
        l0 = opt.launch_count()
        for _ in range(args.steps):
            step_eager()
        torch.cuda.synchronize()
        launches = opt.launch_count() - l0      # kernels per K steps (each replay runs the same set)
        prof = opt.profile_read()
    opt.profile(False)
    stats = opt.stats()
    t = torch.tensor([ms_total], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = 1000.0 / ms_step

    # ---------------- end to end through the public API, host buffers ----------------
    e2e = None
    if not args.no_e2e:
        loss_host = torch.empty(1, dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the host-target gather runs on a side stream overlapped with projection/binning, in a CUDA
        # graph of the step over the pinned host targets (--e2e-mode graph) or launched eagerly
        if gstep is not None and args.e2e_mode == "graph":
            from paper_2506_21117_b200 import GraphStep
            gstep_host = GraphStep(opt, cams, tg_host, n_views_total=V,
                                   allreduce=allreduce_packed if world > 1 else None)
            step_host = gstep_host.replay
        else:
            step_host = (lambda: step_eager(tg_host)) if gstep is not None else (lambda: step(tg_host))
        for _ in range(max(args.warmup, 3)):   # untimed warm-up of this form of the step, like the device-target one
            step_host()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        w0 = time.perf_counter()
        f0.record(stream)
        for k in range(args.steps):
            # this step's inputs: the views' target images stay in pinned host memory; the library
            # moves only the pixels of the active tiles to the device (k_gather_targets, overlapped)
            ev[k].record(stream)
            loss = step_host()
            loss_host.copy_(loss, non_blocking=True)         # the step's result
        ev[args.steps].record(stream)
        f1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        per_step = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps))
        te = torch.tensor([f0.elapsed_time(f1), wall * 1e3], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        st_e = opt.stats()
        h2d = torch.tensor([float(st_e["n_items"]) * 256 * 3 * tbytes], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(h2d)
        e2e = {"value": 1000.0 * args.steps / float(te[1].item()), "unit": "steps/s",
               "h2d_bytes_per_step": int(h2d.item()), "d2h_bytes_per_step": 4 * world,
               "h2d_note": f"target pixels of the active tiles only (256 px x 3 ch x {tbytes} B per active tile), "
                           "read from pinned host memory inside the step; the full target set is "
                           f"{int(tg_host.numel() * tbytes) * world} B",
               "device_ms_per_step": float(te[0].item()) / args.steps,
               "device_step_ms_min_median_max": [round(per_step[0], 4), round(per_step[len(per_step) // 2], 4),
                                                 round(per_step[-1], 4)],
               "mode": ("CUDA graph of the step over the pinned host targets"
                        if gstep is not None and args.e2e_mode == "graph" else "eager launches")}

    # ---------------- end to end with fp32 target images (the BASELINE configs' own format) --------------
    e2e_f32 = None
    if not args.no_e2e and world == 1 and args.targets == "u8" and gstep is not None:
        tg32 = torch.from_numpy(np.ascontiguousarray(sc.targets[my_views], dtype=np.float32)).pin_memory()
        g32 = GraphStep(opt, cams, tg32, n_views_total=V)
        for _ in range(2):
            g32.replay()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            loss = g32.replay()
            loss_host.copy_(loss, non_blocking=True)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        st_f = opt.stats()
        e2e_f32 = {"value": round(1000.0 * args.steps / (wall * 1e3), 3), "unit": "steps/s",
                   "h2d_bytes_per_step": int(st_f["n_items"]) * 256 * 3 * 4, "d2h_bytes_per_step": 4,
                   "note": "same step, target images as fp32 in pinned host memory (the configs' U[0,1] floats)"}
        del g32

    # ---------------- local / full: the same step with every tile active ("w/o Kernel") ----------
    local_full = None
    if world == 1 and not args.all_tiles and not args.no_local_full:
        lim_f = limits_for(args.config, sc.n, len(cams), W, H, True)
        pf = GaussianParams.from_scene(sc, device=f"cuda:{local}")
        of = LocalOptimizer(pf, sc.regions, limits=lim_f)
        if not args.no_spatial_order:
            of.spatial_order()
        for _ in range(2):
            of.forward(cams, tg, n_views_total=V, all_tiles=True)
            of.adam(of.backward())
        torch.cuda.synchronize()
        n_full = 3
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(n_full):
            of.forward(cams, tg, n_views_total=V, all_tiles=True)
            of.adam(of.backward())
        a1.record(stream)
        torch.cuda.synchronize()
        full_ms = a0.elapsed_time(a1) / n_full
        of.close()
        del pf, of
        torch.cuda.empty_cache()
        local_full = {"full_ms_per_step": round(full_ms, 4), "local_ms_per_step": round(ms_step, 4),
                      "ratio": round(ms_step / full_ms, 4),
                      "note": "local = this line's step (masked, static cache, graph); full = every tile active "
                              "(eager, uncached): the P:347 'w/o Kernel' analogue; the paper's Table 13 ratio is "
                              "0.34 at 30% of the tiles (P:528)"}

    out = None
    if rank == 0:
        peaks = _peaks()
        hbm = peaks.get("hbm_gbs", 6650.0)   # fallback: B200_PROFILING.md
        clocks = clk.summary()
        per = {k: v for k, v in prof.items() if v["calls"]}
        dom = max(per, key=lambda k: per[k]["ms"]) if per else None
        step_ms_sum = sum(v["ms"] for v in per.values())
        work = algorithmic_work(sc, len(cams), stats,
                                tiles=(bool(args.static_cache) and not os.environ.get("CLS_NO_TL")) and
                                ("sort" if os.environ.get("CLS_TL_SORT") else "direct"))
        groups = {}
        for k, v in per.items():
            avg_ms = v["ms"] / v["calls"]
            w = work.get(k)
            if w is None:
                continue
            kind, amount = w
            rate = amount / (avg_ms * 1e-3)
            groups[k] = {"ms": round(avg_ms, 4), "bound": kind,
                         ("GB/s" if kind == "hbm" else "TFLOP/s"): round(rate / (1e9 if kind == "hbm" else 1e12), 2)}
        roof = None
        if dom is not None and dom in work:
            kind, amount = work[dom]
            avg_ms = per[dom]["ms"] / per[dom]["calls"]
            if kind == "alu":
                sm_mhz = peaks.get("sm_max_mhz", 1965.0)
                peak = SM_COUNT * FP32_LANES * 2 * sm_mhz * 1e6 / 1e12
                ach = amount / (avg_ms * 1e-3) / 1e12
                roof = {"kernel": dom, "bound": "alu", "achieved": round(ach, 3), "peak": round(peak, 2),
                        "unit": "TFLOP/s", "frac": round(ach / peak, 4), "traffic": None,
                        "peak_source": f"FP32 FMA lanes 148x128x2 at sm_max {sm_mhz:.0f} MHz (MEASURED_PEAKS.json clock)",
                        "units_per_launch": int(stats["n_fwd_evals"] if dom == "fwd_raster" else stats["n_bwd_evals"]),
                        "unit_name": "(pixel, entry) evaluations"}
            else:
                ach = amount / (avg_ms * 1e-3) / 1e9
                roof = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": None,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)", "bytes_per_launch": int(amount)}
            roof["share_of_step"] = round(per[dom]["ms"] / max(step_ms_sum, 1e-9), 3)
            tr = ncu_traffic(args.config, dom)
            if tr is not None and world == 1 and not args.all_tiles:
                roof["traffic"] = tr["bytes"]
                roof["traffic_source"] = f"dram__bytes_read.sum + dram__bytes_write.sum, {tr['source']}"
        # the raster kernels against FP32, MUFU and HBM (BASELINE metric: "raster HBM GB/s vs B200 peak")
        raster = {}
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        fp32_peak = SM_COUNT * FP32_LANES * 2 * sm_mhz * 1e6
        mufu_peak = SM_COUNT * 16 * sm_mhz * 1e6      # ex2 per SM per clock (~4.6 T/s)
        for grp, evals_key, flops in (("fwd_raster", "n_fwd_evals", FWD_FLOPS_PER_EVAL),
                                      ("bwd_raster", "n_bwd_evals", BWD_FLOPS_PER_EVAL)):
            if grp not in per:
                continue
            t_s = per[grp]["ms"] / per[grp]["calls"] * 1e-3
            ev = float(stats[evals_key])
            r = {"ms": round(t_s * 1e3, 4), "evaluations": int(ev),
                 "fp32_tflops": round(ev * flops / t_s / 1e12, 3), "fp32_frac": round(ev * flops / t_s / fp32_peak, 4),
                 "ex2_per_s": round(ev / t_s / 1e12, 3), "mufu_frac": round(ev / t_s / mufu_peak, 4)}
            tr = ncu_traffic(args.config, grp)
            if tr is not None and world == 1 and not args.all_tiles:
                gbs = tr["bytes"] / t_s / 1e9
                r.update({"hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4), "hbm_peak": hbm,
                          "hbm_source": f"ncu dram bytes per launch ({tr['source']}) / this run's event time"})
            if grp == "fwd_raster" and stats.get("n_fwd_exec"):
                # the (pixel, entry) evaluations executed: a warp walks on until all its pixels terminated;
                # the roofline's unit stays the tile-list evaluation of SURVEY §8(d)
                r["executed_evaluations"] = int(stats["n_fwd_exec"])
                r["executed_frac"] = round(stats["n_fwd_exec"] / max(ev, 1.0), 4)
            raster[grp] = r
        out = {
            "metric": "local-opt steps/s (fwd+bwd+masked Adam)",
            "value": round(value, 4), "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "impl": "ours",
            "config": workload_config(args, sc, world, n_active0),
            "row_order": "generator order" if args.no_spatial_order else "Morton (cls_spatial_order at load)",
            "targets_read": "active tiles' pixels only (gathered per active tile)",
            "mpix_per_s": {"rendered": round(sum(stats["n_active_tiles"]) * 256 * world * value / 1e6, 2),
                           "frame_equivalent": round(V * W * H * value / 1e6, 2)},
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "clocks": clocks,
            "step_mode": (f"CUDA graph replay (kernel breakdown from K eager steps; e2e {args.e2e_mode})" if gstep is not None
                          else (graph_note or "eager")),
            "cold_step_ms": round(cold_ms, 4),
            "raster": raster,
            "local_full": local_full,
            "e2e_f32_targets": e2e_f32,
            "static_cache": ({"records": int(stats["cache_records"]), "units": int(stats["cache_units"]),
                              "rows_per_step": int(stats["cache_rows"]), "builds": int(stats["cache_builds"]),
                              "note": "warm steps timed; cold_step_ms = an eager step that rebuilds the cache"}
                             if args.static_cache and not args.all_tiles else None),
            "kernels_ms_per_step": {k: round(v["ms"] / args.steps, 4) for k, v in per.items()},
            "kernel_rates": groups,
            "counts": {k: stats[k] for k in ("n_records", "n_pairs", "n_items", "max_list", "n_units",
                                             "n_fwd_evals", "n_fwd_exec", "n_bwd_evals", "n_candidates", "n_kept_pairs", "n_stage1", "n_tested", "n_live_units")},
        }
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(sc, args.cpu_views)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    opt.close()
    return out


# kernel names of the profile groups in the ncu captures committed under profiles/
# the kernel names in the ncu summaries (with the static cache's exact tile lists the raster kernels
# carry the TL template argument; the uncached names are the fallback)
GROUP_KERNELS = {"fwd_raster": ("k_fwd<1, 0, 1>", "k_fwd<1, 0, 0>", "k_fwd<1, 0>"),
                 "project_cand": ("k_project_cand<1>",), "project_exact": ("k_project_exact<3>",),
                 "bwd_raster": ("k_bwd<1>", "k_bwd<0>", "k_bwd"), "emit": ("k_units",), "bin_count": ("k_permute",)}


def ncu_traffic(config: str, group: str):
    """DRAM bytes per launch of the group's kernel from the newest committed ncu --set full capture of
    this workload (profiles/r*_<config>_ncu_traffic.json), or None."""
    import glob
    import re

    def version(path):   # r<round>_v<n>_... or r<round>_final_...: newest = highest (round, n), final last
        m = re.match(r"r(\d+)_(?:v(\d+)|(final))", os.path.basename(path))
        if not m:
            return (-1, -1)
        return (int(m.group(1)), 1 << 30 if m.group(3) else int(m.group(2)))

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{config}_ncu_traffic.json")), key=version)
    if not files or group not in GROUP_KERNELS:
        return None
    try:
        table = json.load(open(files[-1]))
        rec = next((table[k] for k in GROUP_KERNELS[group] if k in table), None)
        return None if rec is None else {"bytes": int(rec["dram_bytes"]), "source": os.path.basename(files[-1])}
    except Exception:
        return None


def algorithmic_work(sc, n_views, st, tiles=False):
    """Per-launch algorithmic work of each kernel group: bytes the method must
    move for the HBM-bound groups, FP32 FLOPs for the compositing kernels."""
    n, V = sc.n, n_views
    K4 = -(-3 * (sc.sh_degree + 1) ** 2 // 4)
    A, R, P = st["n_active"], st["n_records"], st["n_pairs"]
    C = st.get("n_candidates", R)
    U = st.get("n_units", P)
    rbits = 31 + max(V - 1, 1).bit_length()            # (view, depth) bits above the carried record id
    rpasses = -(-rbits // (8 if rbits <= 32 else 9))
    TY = -(-sc.height // 16)
    upasses = -(-max(V * TY, 1).bit_length() // 8)      # row segments (view, tile row), 8-bit digits
    tbits = max(V * TY * (-(-sc.width // 16)), 1).bit_length()   # tiles (view, tile row, column)
    tpasses = -(-tbits // (8 if tbits <= 16 else 9))
    return {
        "member": ("hbm", n * 16 + n * 4 + A * 4),
        "project_cand": ("hbm", n * 48 + C * 8),
        "project_exact": ("hbm", C * 8 + R * (48 + 16 * K4 + 64 + 4 + 4 + 8)),   # record, gid, rows, key
        "rec_sort": ("hbm", rpasses * R * 16),          # key-only passes: read + write 8 B
        # k_permute: key 8 + rrows 4 in, srid 4 + rcnt 4 out; scan: 4 + 4
        "bin_count": ("hbm", R * (20 + 8)),
        # k_units: per record roff, rcnt, srid, key (20 B) + the 64 B record; per unit the row-mask
        # word (4 B) and the 8 B key out
        "emit": ("hbm", R * (20 + 64) + U * (4 + 8)),
        # key-only passes (record id packed in the key); with the static cache's exact tile lists (k_tiles.cu)
        # the step's units are cut into (tile, record) pairs instead: count (8 in, 4 out), scan (4 + 4),
        # emit (8 + 4 in, 8 out per pair), the key-only pair sort by tile, item ranges + merge keys
        # (8 in, 4 dpos, 8 out per pair).  Direct lists (default): the records' row counts scanned (4 + 4), two
        # passes over the records (64 B each) and their units' row-mask words, a 4 B count per pair, the tiles'
        # scan (4 + 4 per tile), 4 + 8 + 4 B per placed pair, then the per-tile order: 8 + 4 in, 4 rank
        # position, 8 out per pair
        "pair_sort": ("hbm", (R * 8 + 2 * (R * 64 + U * 4) + P * 4 + V * TY * (-(-sc.width // 16)) * 8 + P * 16 +
                              P * 24) if tiles == "direct" else
                      (U * 28 + P * 8 + tpasses * P * 16 + P * 20) if tiles else (upasses * U * 16 + U * 8)),
        "fwd_raster": ("alu", st["n_fwd_evals"] * FWD_FLOPS_PER_EVAL),
        "bwd_raster": ("alu", st["n_bwd_evals"] * BWD_FLOPS_PER_EVAL),
        "bwd_project": ("hbm", A * V * 48 + A * (48 + 16 * K4) + A * 16 * (3 + K4)),
        "adam": ("hbm", A * 16 * (3 + K4) * 7),
    }


def cpu_baseline(sc, n_views):
    """The oracle (as it stands) on a bounded sample: the first `n_views` views of the workload
    (all Gaussians projected, fwd + bwd over their active tiles) plus the masked Adam of the
    active rows, timed on the host cores and scaled to the whole step (x V / n_views)."""
    import oracle
    sub = synth.Scene(sc.name, sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh, sc.sh_degree,
                      sc.cameras[:n_views], sc.regions, sc.targets[:n_views])
    t0 = time.perf_counter()
    fb = oracle.forward_backward(sub, n_views_total=len(sc.cameras))
    rows = oracle.pack_rows(fb["grad"][fb["idx"]], sc.sh_degree)
    lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
    oracle.adam_rows(np.zeros_like(rows), np.zeros_like(rows), np.zeros_like(rows), rows, lr, step=1)
    dt = time.perf_counter() - t0
    V = len(sc.cameras)
    step_s = dt * V / n_views
    return {"value": round(1.0 / step_s, 6), "unit": "steps/s", "cores": oracle.num_threads(), "kind": "oracle",
            "extrapolated": V / n_views != 1, "scale": V / n_views,
            "sample": f"{n_views} of {V} views ({sc.n} Gaussians projected, fwd+bwd over active tiles) + masked "
                      f"Adam; {dt:.2f} s measured, EXTRAPOLATED x{V / n_views:g} to one step"}


def bench_scene(args):
    """The workload's scene; with --targets u8 (default) its targets are 8-bit images (as captured)
    and every consumer -- the kernels through CLS_FLAG_TARGETS_U8, the oracle's cpu baseline and the
    reference arm -- sees the same fp32 values k / 255."""
    sc = synth.make_scene(args.config)
    if args.targets != "u8":
        return sc, None
    u8 = np.floor(np.asarray(sc.targets, np.float64) * 255.0 + 0.5).clip(0, 255).astype(np.uint8)
    return dataclasses.replace(sc, targets=u8.astype(np.float32) / np.float32(255.0)), u8


def workload_config(args, sc, world: int, n_active: int) -> dict:
    """The workload both arms report (`config`): the same dict for `--impl ours` and `--impl reference`."""
    return {"workload": args.config, "gaussians": sc.n, "views": len(sc.cameras), "width": sc.width,
            "height": sc.height, "sh_degree": sc.sh_degree, "active": n_active,
            "mode": "all-tiles (w/o kernel)" if getattr(args, "all_tiles", False) else "masked (local kernel)",
            "parallelism": f"views/dp{world}",
            "targets": "u8 8-bit images (k / 255 in fp32)" if args.targets == "u8" else "fp32",
            "l2": f"inputs larger than L2 (params+moments {sc.n * (12 + 3 * 4 * 4) * 4 * 3 / 1e9:.2f} GB)"}


def run_reference(args):
    """Reference arm = the CPU oracle as it stands, on this arm's config and metric."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    import oracle
    sc, _ = bench_scene(args)
    V = len(sc.cameras)
    sub = synth.Scene(sc.name, sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh, sc.sh_degree,
                      sc.cameras[:1], sc.regions, sc.targets[:1])
    times = []
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        fb = oracle.forward_backward(sub, n_views_total=V)
        rows = oracle.pack_rows(fb["grad"][fb["idx"]], sc.sh_degree)
        lr = oracle.lr_row(sc.sh_degree, [1e-3] * 6)
        oracle.adam_rows(np.zeros_like(rows), np.zeros_like(rows), np.zeros_like(rows), rows, lr, step=1)
        if k >= args.warmup:
            times.append(time.perf_counter() - t0)
    n_active = int(len(fb["idx"]))             # |O^t|: the whole scene's membership, as in the GPU arm
    step_s = statistics.mean(times) * V          # one sampled view per step, scaled to all V views
    value = 1.0 / step_s
    sample = f"1 of {V} views per step (fwd+bwd+Adam, fp64 oracle), EXTRAPOLATED x{V} to the whole step"
    return {"metric": "local-opt steps/s (fwd+bwd+masked Adam)", "value": round(value, 6), "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 2),
            "sample_ms_per_step": round(statistics.mean(times) * 1e3, 2),   # measured; ms_per_step = this x V
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(args, sc, world, n_active),
            "cpu_baseline": {"value": round(value, 6), "unit": "steps/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": sample, "extrapolated": V != 1, "scale": V},
            "e2e": {"value": round(value, 6), "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_loop(args):
    """BASELINE config 5's batched multi-timestep update as the method runs it: `--steps` local-
    optimisation steps (CUDA-graph replays of the cached step) with sphere pruning of O^t every
    `--prune-every` steps (the scene partitioned into its static prefix first); a prune changes
    the row count, so the step is re-captured after it.  Timed end to end on the device (prunes and
    re-captures included).  --per-set: NEXT-3 per-change-set activation instead of the union."""
    import torch

    from paper_2506_21117_b200 import GaussianParams, GraphStep, LocalOptimizer
    torch.cuda.set_device(0)
    sc, u8 = bench_scene(args)
    V = len(sc.cameras)
    cams = sc.cameras
    params = GaussianParams.from_scene(sc, device="cuda:0")
    lim = limits_for(args.config, sc.n, V, sc.width, sc.height, False)
    opt = LocalOptimizer(params, sc.regions, limits=lim, static_cache=True, per_set=args.per_set)
    opt.spatial_order()
    n_static = opt.partition_static()
    tg = torch.from_numpy(np.ascontiguousarray(u8 if u8 is not None else sc.targets)).cuda()
    for _ in range(args.warmup):            # warm-up steps (the first builds the static cache)
        opt.step(cams, tg)
    torch.cuda.synchronize()
    n0 = params.n
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prunes, removed, captures = 0, 0, 0
    gs = GraphStep(opt, cams, tg)   # the first capture is set-up (its host time is not a step's)
    captures += 1
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        trace = [] if os.environ.get("CLS_LOOP_TRACE") else None   # host phases (diagnostic, stderr)
        for k in range(args.steps):
            t0 = time.perf_counter()
            if k > 0 and k % args.prune_every == 0:
                removed += opt.prune_outside()     # O^t rows whose centre left the spheres
                prunes += 1
                gs = None                          # n changed: the captured step is stale
            t1 = time.perf_counter()
            if gs is None:
                gs = GraphStep(opt, cams, tg)
                captures += 1
            t2 = time.perf_counter()
            loss = gs.replay()
            if trace is not None:
                trace.append((k, round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2),
                              round(1e3 * (time.perf_counter() - t2), 2)))
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if trace is not None:
        print(json.dumps({"loop_ms": round(ms, 2), "host_ms": round(sum(sum(t[1:]) for t in trace), 2),
                          "slow": sorted(trace, key=lambda t: -sum(t[1:]))[:10]}), file=sys.stderr)
    stats = opt.stats()
    # per-kernel breakdown: K eager steps right after (same workload)
    opt.profile(True)
    opt.profile_read()
    for _ in range(min(args.steps, 20)):
        opt.step(cams, tg)
    torch.cuda.synchronize()
    prof = opt.profile_read()
    opt.profile(False)
    kk = min(args.steps, 20)
    out = {"metric": "local-opt steps/s (fwd+bwd+masked Adam), 100-step batched loop with sphere pruning",
           "value": round(1000.0 * args.steps / ms, 3), "unit": "steps/s", "n_gpus": 1, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
           "impl": "ours", "dtype": "f32", "data": "synthetic",
           "config": {"workload": args.config, "gaussians": sc.n, "views": V, "width": sc.width,
                      "height": sc.height, "activation": "per change set (NEXT-3)" if args.per_set else "union",
                      "prune_every": args.prune_every, "n_static": int(n_static), "rows_at_start": int(n0),
                      "rows_at_end": int(params.n)},
           "loop": {"prunes": prunes, "rows_removed": int(removed), "graph_captures": captures,
                    "timed": "device events around the whole loop (prunes and re-captures included)"},
           "active": int(stats["n_active"]), "active_tiles": int(sum(stats["n_active_tiles"])),
           "static_cache": {"builds": int(stats["cache_builds"]), "mask_rebuilds": int(stats["cache_mask_builds"]),
                            "refreshes": int(stats["cache_refreshes"]), "records": int(stats["cache_records"]),
                            "note": "a prune changes only the rows >= n_static: S0 is re-formed and the frozen part "
                                    "kept (refresh) when all frozen rows lie below n_static; the rebuilds follow "
                                    "the active mask"},
           "kernels_ms_per_step": {k: round(v["ms"] / kk, 4) for k, v in prof.items() if v["calls"]},
           "clocks": clk.summary()}
    opt.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=synth.CONFIG_NAMES)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--all-tiles", action="store_true", help="full-frame step (P:347 'w/o Kernel')")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-spatial-order", action="store_true",
                    help="keep the synthetic generator's row order (no cls_spatial_order at load)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-local-full", action="store_true", help="skip the all-tiles (local/full) measurement")
    ap.add_argument("--e2e-mode", default="graph", choices=("graph", "eager"))
    ap.add_argument("--targets", default="u8", choices=("u8", "f32"),
                    help="target images as 8-bit (k / 255, CLS_FLAG_TARGETS_U8) or fp32")
    ap.add_argument("--cpu-views", type=int, default=1)
    ap.add_argument("--static-cache", dest="static_cache", choices=("auto", "on", "off"), default="auto",
                    help="CLS_FLAG_STATIC_CACHE: frozen rows' records/units built once, reused (DESIGN.md); auto = "
                         "on from 500k Gaussians (below, the cache's extra graph nodes cost more than the "
                         "projection it saves: c1 4251 vs 3605, c2 2113 vs 1962, c3 1196 vs 1447 steps/s)")
    ap.add_argument("--no-static-cache", dest="static_cache", action="store_const", const="off")
    ap.add_argument("--eager", action="store_true",
                    help="launch every kernel per step instead of replaying the step as one CUDA graph (N = 1)")
    ap.add_argument("--loop", action="store_true", help="the multi-step loop with pruning (BASELINE config 5)")
    ap.add_argument("--prune-every", type=int, default=15)
    ap.add_argument("--per-set", action="store_true", help="NEXT-3 per-change-set activation (with --loop)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.loop and args.impl == "ours":
        out = run_loop(args)
    else:
        out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
