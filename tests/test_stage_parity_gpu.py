"""Stage parity: the records of the projection and the per-tile depth-ordered
lists of the binning, against the oracle's projection of the same inputs -- with and without the static
cache.  Records: every GPU record is a non-culled (view, Gaussian) of the oracle whose rect reaches an
active tile; u, v, conic, colour and opacity agree; the GPU's emission rect lies inside the oracle's
3-sigma rect (R8).  Lists: each sampled active tile's GPU list is an in-order subsequence of the
oracle's rect list in (kappa, index) order (R13, R14) and holds every Gaussian whose fp64 alpha reaches
1/255 (with a 1e-4 margin) at a pixel of the tile (the raster's alpha-footprint culling drops only the
others)."""
import numpy as np
import pytest

import oracle
import synth
from tests import gpu_helpers as H

pytestmark = pytest.mark.gpu

KAPPA = 0.72134752044448170368


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


SCENES = {
    "c2r": lambda: synth.make_scene("c2", n=20000, width=296, height=232, n_views=2),
    "c3s": lambda: synth.make_scene("c3", n=150000, n_views=2),
    "coplanar": lambda: synth.coplanar_scene(),
}


def _run(sc, cached):
    from paper_2506_21117_b200 import GaussianParams, LocalOptimizer, default_limits
    p = GaussianParams.from_scene(sc)
    opt = LocalOptimizer(p, sc.regions, limits=default_limits(sc.n, len(sc.cameras), sc.width, sc.height),
                         static_cache=cached)
    res = opt.forward(sc.cameras, None, images=False, tile_mask=True)
    return opt, res.tile_mask.cpu().numpy().astype(bool)


@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("name", list(SCENES))
def test_record_stage_parity(torch_cuda, name, cached):
    sc = SCENES[name]()
    opt, mask = _run(sc, cached)
    rec, gid, view, count = opt.debug_records(4_000_000)
    dil = int(opt.stats()["cache_dilation"]) if cached else 0
    opt.close()
    assert count == len(gid) and count > 0
    assert len(set(zip(view.tolist(), gid.tolist()))) == count, "one record per (view, Gaussian)"
    for v in range(len(sc.cameras)):
        pr = oracle.project(sc, v)
        sel = view == v
        g = gid[sel]
        r = rec[sel].astype(np.float64)
        assert np.all(pr["culled"][g] == 0), "a record of a culled Gaussian"
        u = r[:, 0] + r[:, 1]
        vv = r[:, 2] + r[:, 3]
        assert np.allclose(u, pr["uv"][g, 0], rtol=0, atol=1e-5 * np.maximum(1.0, np.abs(pr["uv"][g, 0])))
        assert np.allclose(vv, pr["uv"][g, 1], rtol=0, atol=1e-5 * np.maximum(1.0, np.abs(pr["uv"][g, 1])))
        a1, a2, b1, b2 = r[:, 4], r[:, 5], r[:, 6], r[:, 7]
        ca, cb, cc = (a1 * a1 + b1 * b1) / KAPPA, (a1 * a2 + b1 * b2) / KAPPA, (a2 * a2 + b2 * b2) / KAPPA
        oc = pr["conic"][g]
        scale = np.maximum(np.abs(oc[:, 0]), np.abs(oc[:, 2]))
        for got, want in ((ca, oc[:, 0]), (cb, oc[:, 1]), (cc, oc[:, 2])):
            assert np.all(np.abs(got - want) <= 1e-5 * scale)
        assert np.allclose(r[:, 8:11], pr["rgb"][g], rtol=0, atol=1e-5)
        assert np.allclose(r[:, 11], pr["opac"][g], rtol=1e-6, atol=0)
        rx = np.ascontiguousarray(rec[sel][:, 14]).view(np.int32)   # rect corners ride as int bits
        ry = np.ascontiguousarray(rec[sel][:, 15]).view(np.int32)
        x0, y0, x1, y1 = rx & 0xffff, rx >> 16, ry & 0xffff, ry >> 16
        orc = pr["rect"][g]
        assert np.all((x0 >= orc[:, 0]) & (y0 >= orc[:, 1]) & (x1 <= orc[:, 2]) & (y1 <= orc[:, 3]))
        assert np.all((x1 > x0) & (y1 > y0))
        # each record's rect reaches an active tile (cached frozen records: a tile of the dilated mask
        # they were built against, the active rects grown by the build's dilation)
        m = mask[v]
        if cached:
            assert dil >= 1
            mp = np.pad(m, dil)
            m = np.zeros_like(m)
            for dy in range(2 * dil + 1):
                for dx in range(2 * dil + 1):
                    m |= mp[dy:dy + mask.shape[1], dx:dx + mask.shape[2]]
        for k in range(0, len(g), max(1, len(g) // 400)):
            assert m[y0[k]:y1[k], x0[k]:x1[k]].any()


def _max_alpha_on_tile(pr, idx, tx, ty, W, H):
    xs = np.arange(tx * 16, min(tx * 16 + 16, W), dtype=np.float64)
    ys = np.arange(ty * 16, min(ty * 16 + 16, H), dtype=np.float64)
    X, Y = np.meshgrid(xs, ys)
    out = np.zeros(len(idx))
    for j, i in enumerate(idx):
        dx = pr["uv"][i, 0] - X
        dy = pr["uv"][i, 1] - Y
        a, b, c = pr["conic"][i]
        p = -0.5 * (a * dx * dx + c * dy * dy) - b * dx * dy
        al = np.where(p <= 0.0, pr["opac"][i] * np.exp(np.minimum(p, 0.0)), 0.0)
        out[j] = min(0.99, al.max())
    return out


@pytest.mark.parametrize("cached", [False, True])
@pytest.mark.parametrize("name", list(SCENES))
def test_tile_list_stage_parity(torch_cuda, name, cached):
    sc = SCENES[name]()
    opt, mask = _run(sc, cached)
    rng = np.random.default_rng(5)
    TX, TY = -(-sc.width // 16), -(-sc.height // 16)
    checked = 0
    for v in range(len(sc.cameras)):
        pr = oracle.project(sc, v)
        live = np.nonzero(pr["culled"] == 0)[0]
        rc = pr["rect"][live]
        tiles = np.nonzero(mask[v].reshape(-1))[0]
        for t in rng.choice(tiles, size=min(12, len(tiles)), replace=False):
            tx, ty = int(t % TX), int(t // TX)
            inr = (rc[:, 0] <= tx) & (tx < rc[:, 2]) & (rc[:, 1] <= ty) & (ty < rc[:, 3])
            cand = live[inr]
            order = np.lexsort((cand, pr["depth_key"][cand]))     # (kappa, index), R13
            cand = cand[order]
            gpu = opt.debug_tile_list(v, int(t))
            pos = {int(g): k for k, g in enumerate(cand)}
            assert all(int(g) in pos for g in gpu), "GPU list entry outside the oracle's rect list"
            ks = [pos[int(g)] for g in gpu]
            assert ks == sorted(ks) and len(set(ks)) == len(ks), "GPU list order differs from (kappa, index)"
            amax = _max_alpha_on_tile(pr, cand, tx, ty, sc.width, sc.height)
            required = set(int(g) for g in cand[amax >= (1.0 / 255.0) * (1.0 + 1e-4)])
            assert required <= set(int(g) for g in gpu), "a Gaussian reaching alpha >= 1/255 is missing"
            checked += 1
    opt.close()
    assert checked > 0
