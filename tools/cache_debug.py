"""Diagnostics of the static cache: cached vs uncached step on one scene, step by step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def run(sc, steps, cached, lr=1e-3):
    import torch
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height),
                         lr=(lr,) * 6, static_cache=cached)
    tg = torch.from_numpy(np.ascontiguousarray(sc.targets)).cuda()
    out = []
    for k in range(steps):
        res = opt.forward(sc.cameras, tg, images=True, tile_mask=True)
        g = opt.backward()
        opt.adam(g)
        torch.cuda.synchronize()
        out.append((res.images.cpu().numpy(), res.tile_mask.cpu().numpy(), opt.stats()))
    opt.close()
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3s"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    sc = {"c2r": lambda: synth.make_scene("c2", n=20000, width=296, height=232, n_views=2),
          "c3s": lambda: synth.make_scene("c3", n=150000, n_views=2),
          "c1": lambda: synth.make_scene("c1")}[name]()
    a = run(sc, steps, False)
    b = run(sc, steps, True)
    for k in range(steps):
        ia, ib = a[k][0], b[k][0]
        d = np.abs(ia - ib).max(axis=1)
        print(f"step {k}: differing px {int((d > 0).sum())} max {float(d.max()):.3g} mask eq {np.array_equal(a[k][1], b[k][1])}")
        for v in range(d.shape[0]):
            ys, xs = np.nonzero(d[v] > 0)
            if ys.size:
                tiles = sorted(set(zip((ys // 16).tolist(), (xs // 16).tolist())))
                print(f"  view {v}: {ys.size} px in {len(tiles)} tiles, first {tiles[:6]}")
        sa, sb = a[k][2], b[k][2]
        keys = ["n_active", "n_records", "n_items", "n_units", "n_live_units", "n_pairs", "n_fwd_evals", "max_list",
                "cache_mode", "cache_valid", "cache_builds", "cache_records", "cache_units", "cache_rows", "overflow"]
        print("  uncached", {x: sa[x] for x in keys})
        print("  cached  ", {x: sb[x] for x in keys})


if __name__ == "__main__":
    main()
