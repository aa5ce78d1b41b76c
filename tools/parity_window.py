"""Measure the fp32 error of the CUDA path's compositing decisions against the fp64 oracle, to set
the parity protocol's ambiguity window from data.

For every pixel of an active tile: the oracle's T_final, composited count K and path sums
S1 = sum r_j, S2 = sqrt(sum r_j^2) (r_j = alpha_j / (1 - alpha_j)); the GPU's T_final
(cls_debug_pixels).  A pixel whose decisions agree has |dT|/T << 1/255 (one skipped or terminated
Gaussian changes T by a factor (1 - alpha) with alpha >= 1/255), so pixels with |dT|/T < 1e-3 give
the error distribution of fp32 T; pixels with K = 1 give that of fp32 alpha (T = 1 - alpha).
Candidate windows are then scored: ambiguous fraction of compared pixels, and pixels off by more
than 1e-4 that the window does NOT flag (must be 0).

    python tools/parity_window.py [--out gpurun_out/parity_window.json] [--scenes c1,c2r,...]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: a diagnostics tool, not the product path)
import synth  # noqa: E402


def scenes(names):
    out = {}
    for nm in names:
        if nm == "c1":
            out[nm] = synth.make_scene("c1")
        elif nm == "c2r":
            out[nm] = synth.make_scene("c2", n=20000, width=296, height=232, n_views=2)
        elif nm == "c2":
            out[nm] = synth.make_scene("c2")
        elif nm == "c3s":
            out[nm] = synth.make_scene("c3", n=150000, n_views=2)
        elif nm == "c3":
            out[nm] = synth.make_scene("c3")
        elif nm == "c5s":
            out[nm] = synth.make_scene("c5", n=150000, n_views=5)
        elif nm == "c4":
            sc = synth.make_scene("c4")
            v = [0, 1]
            out[nm] = synth.Scene(sc.name, sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh,
                                  sc.sh_degree, [sc.cameras[i] for i in v], sc.regions, sc.targets[v])
        elif nm == "coplanar":
            out[nm] = synth.coplanar_scene()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/parity_window.json")
    ap.add_argument("--scenes", default="c1,c2r,c3s,c5s,coplanar,c2,c4")
    a = ap.parse_args()
    import torch
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    res = {}
    margins_bad = []
    # reference window for the margins: the survey's delta = 1e-5 on alpha, the linear T bound
    W1 = (1e-5, 1e-5, 2.0 ** -24)
    all_rT, all_S1, all_S2, all_K, all_da = [], [], [], [], []
    rows = {}
    for nm, sc in scenes(a.scenes.split(",")).items():
        t0 = time.time()
        p = GaussianParams.from_scene(sc)
        opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height))
        r = opt.forward(sc.cameras, None, images=True)
        Tg = opt.debug_pixels().cpu().numpy().astype(np.float64)
        img = r.images.cpu().numpy().astype(np.float64)
        torch.cuda.synchronize()
        opt.close()
        per = []
        for v in range(len(sc.cameras)):
            o = oracle.render(sc, v, oracle.membership(sc), with_grad=False, use_target=False, window=(0.0, 0.0, 0.0))
            comp = np.kron(o["tile_mask"], np.ones((16, 16), bool))[: sc.height, : sc.width]
            To, K, S1, S2 = o["T_final"], o["n_contrib"], o["path"][..., 0], o["path"][..., 1]
            ow = oracle.render(sc, v, oracle.membership(sc), with_grad=False, use_target=False, window=W1)
            rT = np.abs(Tg[v] - To) / np.maximum(To, 1e-30)
            dimg = np.abs(img[v] - o["image"]).max(axis=0)
            same = comp & (rT < 1e-3)
            all_rT.append(rT[same]); all_S1.append(S1[same]); all_S2.append(S2[same]); all_K.append(K[same])
            one = same & (K == 1)
            al = 1.0 - To[one]
            all_da.append(rT[one] * To[one] / np.maximum(al, 1e-30))   # |d alpha| / alpha
            bad = comp & (dimg > 1e-4)
            mg = ow["path"][..., 2]
            margins_bad.append(mg[bad])
            per.append(dict(view=v, compared=int(comp.sum()), flipped=int((comp & (rT >= 1e-3)).sum()),
                            bad_1e4=int(bad.sum()), max_K=int(K.max()),
                            max_margin_bad=float(mg[bad].max()) if bad.any() else None))
            rows.setdefault(nm, []).append((sc, v, comp, dimg))
        res[nm] = dict(views=per, seconds=round(time.time() - t0, 1))
        print(nm, per, flush=True)
    # alpha probe: the c4 scene thinned to isolated splats (same size / opacity / camera distributions),
    # every tile rendered; pixels with ONE composited Gaussian give |d alpha| / alpha = |dT| (1 - alpha)... /
    # alpha directly, over millions of samples (the tail alpha < 0.05 is where the skip test decides)
    probe = dict(all=[], tail=[])
    if "c4" in a.scenes.split(","):
        sc4 = synth.make_scene("c4")
        rng = np.random.default_rng(77)
        keep = np.sort(rng.choice(sc4.n, 30000, replace=False))
        views = [0, 1, 2, 3]
        thin = synth.Scene("c4thin", sc4.means[keep], sc4.log_scales[keep], sc4.quats[keep],
                           sc4.opacity_logits[keep], sc4.sh[keep], sc4.sh_degree, [sc4.cameras[v] for v in views],
                           sc4.regions, None)
        p = GaussianParams.from_scene(thin)
        opt = LocalOptimizer(p, thin.regions, limits=default_limits(thin.n, len(views), thin.width, thin.height))
        opt.forward(thin.cameras, None, images=False, all_tiles=True)
        Tg = opt.debug_pixels().cpu().numpy().astype(np.float64)
        torch.cuda.synchronize()
        opt.close()
        for v in range(len(views)):
            o = oracle.render(thin, v, np.zeros(thin.n, bool), with_grad=False, use_target=False, all_tiles=True,
                              window=(0.0, 0.0, 0.0))
            To, K = o["T_final"], o["n_contrib"]
            one = (K == 1) & np.isfinite(Tg[v])
            one &= np.abs(Tg[v] - To) < 1e-3 * To          # no flip (a flip moves T by >= 1/255)
            al = 1.0 - To[one]
            rel = np.abs(Tg[v][one] - To[one]) / np.maximum(al, 1e-30)   # |d alpha| / alpha (T = 1 - alpha)
            probe["all"].append(rel)
            probe["tail"].append(rel[al < 0.05])
    pa = np.concatenate(probe["all"]) if probe["all"] else np.zeros(0)
    pt = np.concatenate(probe["tail"]) if probe["tail"] else np.zeros(0)
    rT = np.concatenate(all_rT); S1 = np.concatenate(all_S1); S2 = np.concatenate(all_S2)
    K = np.concatenate(all_K).astype(np.float64); da = np.concatenate(all_da)
    u = 2.0 ** -24
    stats = dict(
        n_pixels=int(rT.size),
        rT_percentiles={q: float(np.percentile(rT, q)) for q in (50, 90, 99, 99.9, 100)},
        dalpha_rel_K1=dict(n=int(da.size), p99=float(np.percentile(da, 99)) if da.size else None,
                           max=float(da.max()) if da.size else None),
        # smallest dt1 with rT <= dt1 S1 + 2 u K on every agreeing pixel (u = 2^-24, one rounding per composite)
        dt1_needed=float(np.max((rT - 2 * u * K) / np.maximum(S1, 1e-12))),
        per_K_max={int(k): float(rT[K == k].max()) for k in (1, 2, 5, 10, 20, 40, 70, 100) if np.any(K == k)},
        rms_ratio_max=float(np.max(rT / np.maximum(S2, 1e-12) * (S2 > 0.05))),
    )
    stats["alpha_probe"] = dict(n=int(pa.size), n_tail=int(pt.size),
                                p99=float(np.percentile(pa, 99)) if pa.size else None,
                                p9999=float(np.percentile(pa, 99.99)) if pa.size else None,
                                max=float(pa.max()) if pa.size else None,
                                tail_p9999=float(np.percentile(pt, 99.99)) if pt.size else None,
                                tail_max=float(pt.max()) if pt.size else None)
    mb = np.concatenate(margins_bad) if margins_bad else np.zeros(0)
    stats["bad_pixels"] = int(mb.size)
    stats["bad_margin_vs_W1"] = dict(window=W1, max=float(mb.max()) if mb.size else None,
                                     p99=float(np.percentile(mb, 99)) if mb.size else None,
                                     p90=float(np.percentile(mb, 90)) if mb.size else None)
    print(json.dumps(stats, indent=1), flush=True)
    # candidate windows: (da, dt1, dtk)
    da_m = stats["dalpha_rel_K1"]["max"] or 1e-6
    cands = {"old_linear": (1e-5, 1e-5, 1.2e-7)}
    if pa.size:
        da_m = max(float(pa.max()), da_m)
    for f in (1, 2):
        cands[f"measured_x{f}"] = (f * da_m, f * max(stats["dt1_needed"], 0.0), f * 2 * u)
    if mb.size:   # the window that flags every bad pixel, scaled from W1, with a factor 2 of headroom
        f = 2.0 * float(mb.max())
        cands["bad_margin_x2"] = (f * W1[0], f * W1[1], max(f, 1.0) * W1[2])
    scores = {}
    for cn, w in cands.items():
        tot_c = tot_a = tot_bad = 0
        per = {}
        for nm, lst in rows.items():
            sc_c = sc_a = sc_b = 0
            for sc, v, comp, dimg in lst:
                o = oracle.render(sc, v, oracle.membership(sc), with_grad=False, use_target=False, window=w)
                amb = o["ambiguous"] & comp
                sc_c += int(comp.sum()); sc_a += int(amb.sum()); sc_b += int((comp & ~amb & (dimg > 1e-4)).sum())
            per[nm] = dict(compared=sc_c, ambiguous=sc_a, frac=sc_a / max(sc_c, 1), unflagged_bad=sc_b)
            tot_c += sc_c; tot_a += sc_a; tot_bad += sc_b
        scores[cn] = dict(window=w, per_scene=per, frac=tot_a / max(tot_c, 1), unflagged_bad=tot_bad)
        print(cn, json.dumps(scores[cn]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(dict(scenes=res, stats=stats, candidates=scores), f, indent=1)


if __name__ == "__main__":
    main()
