"""Pins of the CPU oracle against things other than itself (closed forms,
invariants, special cases, finite differences, scipy).  No GPU needed.

Each test names the pin of DESIGN.md §Oracle pins it implements (P1..P14,
V1..V4) and the paper passage the property comes from.
"""
import math

import numpy as np
import pytest

import oracle
import synth

C0 = 0.28209479177387814


def _dc(c):
    """DC SH coefficient giving colour c (R15/R16 closed form: c = C0 f + 1/2)."""
    return (np.asarray(c, np.float64) - 0.5) / C0


def _one_cam(W=64, H=64, f=100.0, cx=32.5, cy=32.5):
    return synth.Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), f, f, cx, cy, W, H)


def _scene(means, ls, quats, ops, sh, deg, cams, regions=None, targets=None):
    if regions is None:
        regions = [synth.Region(synth.REGION_SPHERE, np.zeros(3), np.zeros(3), 1e6)]
    s = synth.scene_from_arrays(means, ls, quats, ops, sh, deg, cams, regions, targets)
    # keep float64 parameters when given (FD harness needs exact perturbations)
    s.means = np.asarray(means, np.float64) if np.asarray(means).dtype == np.float64 else s.means
    return s


# ---------------------------------------------------------------------------
# V1 / P1: single isotropic Gaussian on the optical axis
# ---------------------------------------------------------------------------

def test_v1_single_isotropic_gaussian(oracle_lib):
    cam = _one_cam()
    sc = _scene(np.array([[0.0, 0.0, 2.0]]), np.log([[0.05] * 3]), [[1, 0, 0, 0]], [math.log(4.0)],
                np.full((1, 1, 3), _dc(0.6)), 0, [cam])
    p = oracle.project(sc, 0)
    o = 1.0 / (1.0 + math.exp(-float(np.float32(math.log(4.0)))))
    s = math.exp(float(np.float32(math.log(0.05))))
    sig2 = (100.0 * s / 2.0) ** 2 + 0.3            # (f s / z)^2 + 0.3
    assert p["cov2d"][0] == pytest.approx([sig2, 0.0, sig2], rel=1e-12, abs=1e-12)
    assert p["radius"][0] == 8                      # ceil(3 sqrt(6.866...)) = ceil(7.861)
    assert list(p["rect"][0]) == [1, 1, 3, 3]
    assert p["uv"][0] == pytest.approx([32.0, 32.0], abs=1e-12)
    r = oracle.render(sc, 0, np.ones(1, bool), p, use_target=False, with_grad=False)
    img = r["image"][0]
    c = float(np.float32(_dc(0.6))) * C0 + 0.5
    for d in (0, 1, 3, 5, 8):
        alpha = min(0.99, o * math.exp(-0.5 * d * d / sig2))
        expect = c * alpha if alpha >= 1 / 255 else 0.0
        assert img[32, 32 + d] == pytest.approx(expect, rel=1e-12, abs=1e-15)
    assert img[32, 32 + 9] == 0.0                   # alpha = 0.00165 < 1/255 -> skipped (R2)
    assert img[32, 32] == pytest.approx(0.48, rel=1e-6)         # peak = c min(0.99, o)
    assert r["T_final"][32, 32] == pytest.approx(0.2, rel=1e-6)
    # outside the rect (tiles 1..2) nothing is composited even where alpha would be > 0 (R8)
    assert img[32, 15] == 0.0 and img[32, 48] == 0.0
    # V1 gradient: d C_peak(red) / d opacity_logit = c o (1 - o)
    up = np.zeros((3, 64, 64)); up[0, 32, 32] = 1.0
    r = oracle.render(sc, 0, np.ones(1, bool), p, dL_dC=up)
    g = oracle.backward_project(sc, 0, np.ones(1, bool), p, r["grad2d"])
    assert g[0, 10] == pytest.approx(c * o * (1 - o), rel=1e-10)
    assert abs(c * o * (1 - o) - 0.096) < 1e-6


def test_p1_depth_doubling_quarters_covariance(oracle_lib):
    cam = _one_cam()
    sc = _scene(np.array([[0.0, 0.0, 2.0], [0.0, 0.0, 4.0]]), np.log([[0.05] * 3] * 2), [[1, 0, 0, 0]] * 2,
                [0.0, 0.0], np.zeros((2, 1, 3)), 0, [cam])
    p = oracle.project(sc, 0)
    pre = p["cov2d"][:, [0, 2]] - 0.3
    assert pre[0] == pytest.approx(4.0 * pre[1], rel=1e-12)


# ---------------------------------------------------------------------------
# V2 / V3 / P2: transmittance products and termination
# ---------------------------------------------------------------------------

def _coincident(opacities, colours):
    cam = _one_cam()
    n = len(opacities)
    means = np.array([[0.0, 0.0, 2.0 + 0.5 * k] for k in range(n)])
    ls = np.log(np.full((n, 3), 0.05))
    ops = np.log(np.array(opacities) / (1 - np.array(opacities)))
    sh = _dc(np.array(colours, np.float64)).reshape(n, 1, 3)
    sc = _scene(means, ls, [[1, 0, 0, 0]] * n, ops, sh, 0, [cam])
    sc.opacity_logits = ops.astype(np.float64)
    sc.sh = sh
    sc.log_scales = ls
    return sc


def test_v2_transmittance_product(oracle_lib):
    sc = _coincident([0.5, 0.6, 0.7], [[1, 0, 0], [0, 1, 0], [0, 0, 1]])
    r = oracle.render(sc, 0, np.ones(3, bool), use_target=False, with_grad=False)
    assert r["image"][:, 32, 32] == pytest.approx([0.5, 0.3, 0.14], abs=1e-12)
    assert r["T_final"][32, 32] == pytest.approx(0.06, abs=1e-12)


def test_v3_termination(oracle_lib):
    sc = _coincident([0.98, 0.98, 0.98], [[1, 0, 0], [0, 1, 0], [0, 0, 1]])
    r = oracle.render(sc, 0, np.ones(3, bool), use_target=False, with_grad=False)
    assert r["image"][:, 32, 32] == pytest.approx([0.98, 0.0196, 0.0], abs=1e-12)
    assert r["T_final"][32, 32] == pytest.approx(4e-4, rel=1e-9)
    assert r["n_contrib"][32, 32] == 2


# ---------------------------------------------------------------------------
# V4 / P11: Adam closed form
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("g,expect", [(0.5, [0.999, 0.998, 0.997]),
                                      (-2e-12, [1.0009995002498750, 1.0019990004997501, 1.0029985007496252])])
def test_v4_adam_closed_form(oracle_lib, g, expect):
    th = np.ones((1, 16)); m = np.zeros((1, 16)); v = np.zeros((1, 16))
    lr = oracle.lr_row(0, [1e-3] * 6)
    for step, e in enumerate(expect, start=1):
        th, m, v = oracle.adam_rows(th, m, v, np.full((1, 16), g), lr, step=step)
        # with constant g, m_hat = g and v_hat = g^2 exactly -> step = lr g / (|g| + eps)
        assert th[0, 0] == pytest.approx(e, rel=1e-12)
        assert th[0, 11] == 1.0 and th[0, 15] == 1.0   # pad lanes (scale.w, sh pad) untouched


# ---------------------------------------------------------------------------
# P3 opacity-0 invariance, P4 frozen gradients, P13 A = 0
# ---------------------------------------------------------------------------

def test_p3_zero_opacity_invariance(oracle_lib):
    base = synth.make_scene("c1", n=300)
    fb0 = oracle.forward_backward(base)
    rng = np.random.default_rng(7)
    extra = 50
    sc = synth.make_scene("c1", n=300)
    # extras are frozen (outside the change sphere) so they cannot alter the tile mask (R9)
    pts = rng.uniform(-1, 1, (4 * extra, 3))
    reg = sc.regions[0]
    pts = pts[np.linalg.norm(pts - reg.a.astype(np.float64), axis=1) > reg.r + 1e-3][:extra]
    sc.means = np.concatenate([sc.means, pts.astype(np.float32)])
    sc.log_scales = np.concatenate([sc.log_scales, np.full((extra, 3), -3.0, np.float32)])
    sc.quats = np.concatenate([sc.quats, np.tile(np.float32([1, 0, 0, 0]), (extra, 1))])
    sc.opacity_logits = np.concatenate([sc.opacity_logits, np.full(extra, -30.0, np.float32)])
    sc.sh = np.concatenate([sc.sh, np.zeros((extra, 1, 3), np.float32)])
    fb1 = oracle.forward_backward(sc)
    for r0, r1 in zip(fb0["renders"], fb1["renders"]):
        assert np.array_equal(r0["image"], r1["image"])
    assert np.array_equal(fb0["grad"], fb1["grad"][:300])
    assert np.all(fb1["grad"][300:] == 0.0)


def test_p4_frozen_gradients_exactly_zero(oracle_lib):
    sc = synth.make_scene("c2", n=4000, width=160, height=144, n_views=2)
    fb = oracle.forward_backward(sc)
    act = fb["active"]
    assert act.any() and (~act).any()
    assert np.all(fb["grad"][~act] == 0.0)
    assert np.any(fb["grad"][act] != 0.0)


def test_p13_empty_active_set(oracle_lib):
    sc = synth.make_scene("c1", n=200)
    sc.regions = [synth.Region(synth.REGION_SPHERE, np.array([50.0, 50, 50]), np.zeros(3), 0.1)]
    fb = oracle.forward_backward(sc)
    assert fb["idx"].size == 0
    r = fb["renders"][0]
    assert r["n_active_tiles"] == 0 and not r["tile_mask"].any()
    assert np.all(r["image"] == 0.0) and np.all(r["T_final"] == 1.0)
    assert np.all(fb["grad"] == 0.0) and fb["loss"] == 0.0


def test_p6_empty_scene_black(oracle_lib):
    sc = synth.make_scene("c1", n=100)
    sc.opacity_logits[:] = -40.0
    r = oracle.render(sc, 0, np.ones(sc.n, bool), use_target=False, with_grad=False, all_tiles=True)
    assert np.all(r["image"] == 0.0) and np.all(r["T_final"] == 1.0)


# ---------------------------------------------------------------------------
# P5 exactness and P6 mask neutrality
# ---------------------------------------------------------------------------

def test_p5_exactness_masked_equals_full_frame(oracle_lib):
    sc = synth.make_scene("c2", n=6000, width=208, height=176, n_views=2)
    masked = oracle.forward_backward(sc)
    full = oracle.forward_backward(sc, all_tiles=True)
    act = masked["active"]
    assert 0 < act.sum() < sc.n
    gm, gf = masked["grad"][act], full["grad"][act]
    assert np.abs(gm - gf).max() <= 1e-12 * max(np.abs(gf).max(), 1e-30)
    for rm, rf in zip(masked["renders"], full["renders"]):
        tm = np.kron(rm["tile_mask"], np.ones((16, 16), bool))[: sc.height, : sc.width]
        assert tm.any() and not tm.all()
        assert np.array_equal(rm["image"][:, tm], rf["image"][:, tm])


def test_p6_mask_neutrality(oracle_lib):
    sc = synth.make_scene("c1", n=400)
    act = np.ones(sc.n, bool)                  # every Gaussian active -> every covered tile active
    a = oracle.forward_backward(sc, active=act)
    b = oracle.forward_backward(sc, active=act, all_tiles=True)
    ra, rb = a["renders"][0], b["renders"][0]
    cov = ra["tile_mask"]
    tm = np.kron(cov, np.ones((16, 16), bool))[: sc.height, : sc.width]
    assert np.array_equal(ra["image"][:, tm], rb["image"][:, tm])
    assert np.all(rb["image"][:, ~tm] == 0.0)  # tiles no Gaussian covers are background anyway
    assert np.array_equal(a["grad"], b["grad"])


# ---------------------------------------------------------------------------
# P7 central finite differences (smooth probe loss, Richardson-extrapolated), tiny scenes
# ---------------------------------------------------------------------------

def _f64_scene(sc):
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        setattr(sc, k, np.asarray(getattr(sc, k), np.float64).copy())
    return sc


def _probe(sc, w, act):
    tot, sigs, rects = 0.0, [], []
    for v in range(len(sc.cameras)):
        p = oracle.project(sc, v)
        r = oracle.render(sc, v, act, p, use_target=False, with_grad=False)
        tot += float(np.sum(w[v] * r["image"]))
        sigs.append(r["sig"].copy())
        rects.append((p["rect"].copy(), p["culled"].copy(), p["clamped"].copy()))
    return tot, sigs, rects


def _same_decisions(a, b):
    for sa, sb in zip(a[1], b[1]):
        if not np.array_equal(sa, sb):
            return False
    for (ra, ca, cla), (rb, cb, clb) in zip(a[2], b[2]):
        if not (np.array_equal(ra, rb) and np.array_equal(ca, cb) and np.array_equal(cla, clb)):
            return False
    return True


@pytest.mark.parametrize("seed,deg,views", [(11, 1, 1), (12, 3, 2), (13, 2, 1), (14, 0, 2)])
def test_p7_finite_differences(oracle_lib, seed, deg, views):
    sc = _f64_scene(synth.tiny_scene(seed, n=8, sh_degree=deg, n_views=views))
    act = oracle.membership(sc)
    assert act.all()
    rng = np.random.default_rng(seed + 100)
    w = rng.standard_normal((views, 3, sc.height, sc.width))
    fb = oracle.forward_backward(sc, active=act, dL_dC=w)
    g = fb["grad"]
    eps = 1e-4
    fields = [("means", 3, 0), ("quats", 4, 3), ("log_scales", 3, 7), ("opacity_logits", 1, 10), ("sh", None, 11)]
    checked = rejected = 0
    worst = 0.0
    for i in range(sc.n):
        for name, width, col in fields:
            arr = getattr(sc, name)
            flat = arr[i].reshape(-1) if arr.ndim > 1 else None
            count = width if width is not None else flat.size
            for j in range(count):
                def setv(val):
                    if arr.ndim == 1:
                        arr[i] = val
                    else:
                        view = arr[i].reshape(-1)
                        view[j] = val
                        arr[i] = view.reshape(arr[i].shape)
                x0 = arr[i] if arr.ndim == 1 else arr[i].reshape(-1)[j]
                fds, ok = [], True
                for h in (eps, eps / 2):
                    setv(x0 + h)
                    lp = _probe(sc, w, act)
                    setv(x0 - h)
                    lm = _probe(sc, w, act)
                    setv(x0)
                    ok = ok and _same_decisions(lp, lm)
                    fds.append((lp[0] - lm[0]) / (2 * h))
                if not ok:
                    rejected += 1
                    continue
                fd = (4.0 * fds[1] - fds[0]) / 3.0   # Richardson: removes the O(eps^2) truncation term
                an = g[i, col + j]
                err = abs(fd - an) / max(abs(fd), abs(an), 1e-8)
                worst = max(worst, err)
                checked += 1
                assert err < 1e-5, (name, i, j, fd, an)
    assert checked > 0.9 * (checked + rejected)
    assert worst < 1e-5


# ---------------------------------------------------------------------------
# P8 quaternion scale, P9 principal-point shift, P10 permutation
# ---------------------------------------------------------------------------

def test_p8_quaternion_scale(oracle_lib):
    sc = _f64_scene(synth.tiny_scene(21, n=6, sh_degree=1))
    act = np.ones(sc.n, bool)
    w = np.random.default_rng(3).standard_normal((1, 3, sc.height, sc.width))
    a = oracle.forward_backward(sc, active=act, dL_dC=w)
    lam = 2.5
    sc.quats *= lam
    b = oracle.forward_backward(sc, active=act, dL_dC=w)
    assert np.allclose(a["renders"][0]["image"], b["renders"][0]["image"], rtol=0, atol=1e-14)
    ga, gb = a["grad"][:, 3:7], b["grad"][:, 3:7]
    assert np.allclose(gb * lam, ga, rtol=1e-9, atol=1e-14)
    dots = np.sum(sc.quats * gb, axis=1)
    assert np.all(np.abs(dots) <= 1e-12 * np.abs(gb).sum(axis=1).max() * lam + 1e-18)


def test_p9_principal_point_shift(oracle_lib):
    sc = synth.make_scene("c1", n=500, width=128, height=96)
    act = np.ones(sc.n, bool)
    a = oracle.render(sc, 0, act, use_target=False, with_grad=False, all_tiles=True)
    cam = sc.cameras[0]
    sc.cameras[0] = synth.Camera(cam.R, cam.t, cam.fx, cam.fy, cam.cx + 16.0, cam.cy, cam.width, cam.height)
    b = oracle.render(sc, 0, act, use_target=False, with_grad=False, all_tiles=True)
    assert np.allclose(b["image"][:, :, 16:], a["image"][:, :, :-16], rtol=0, atol=1e-12)


def test_p10_permutation(oracle_lib):
    sc = synth.make_scene("c2", n=3000, width=160, height=160, n_views=1)
    act = oracle.membership(sc)
    a = oracle.forward_backward(sc, active=act)
    perm = np.random.default_rng(5).permutation(sc.n)
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        setattr(sc, k, getattr(sc, k)[perm].copy())
    b = oracle.forward_backward(sc, active=act[perm])
    # the test's depth keys are distinct (checked) so the order is permutation independent
    keys = a["renders"][0]["proj"]["depth_key"][~a["renders"][0]["proj"]["culled"].astype(bool)]
    assert np.unique(keys).size == keys.size
    assert np.array_equal(a["renders"][0]["image"], b["renders"][0]["image"])
    assert np.allclose(a["grad"][perm], b["grad"], rtol=1e-12, atol=1e-300)


# ---------------------------------------------------------------------------
# P12 literal mode == tile-list mode; P14 tile grids
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("cfg,kw", [("c1", {}), ("c2", dict(n=2500, width=144, height=112, n_views=1))])
def test_p12_literal_equals_tile_list(oracle_lib, cfg, kw):
    sc = synth.make_scene(cfg, **kw)
    a = oracle.forward_backward(sc, literal=True)
    b = oracle.forward_backward(sc, literal=False)
    for ra, rb in zip(a["renders"], b["renders"]):
        assert np.array_equal(ra["image"], rb["image"])
        assert np.array_equal(ra["T_final"], rb["T_final"])
        assert np.array_equal(ra["n_contrib"], rb["n_contrib"])
    assert np.array_equal(a["grad"], b["grad"])
    assert a["loss"] == b["loss"]


@pytest.mark.parametrize("wh,grid", [((960, 540), (60, 34)), ((1297, 840), (82, 53)), ((1920, 1080), (120, 68)),
                                     ((128, 128), (8, 8))])
def test_p14_tile_grids(oracle_lib, wh, grid):
    W, H = wh
    sc = synth.make_scene("c1", n=50, width=W, height=H)
    r = oracle.render(sc, 0, np.zeros(sc.n, bool), use_target=False, with_grad=False)
    assert r["tile_mask"].shape == (grid[1], grid[0])


# ---------------------------------------------------------------------------
# membership pins (R21): inclusive boundaries, spheres and boxes
# ---------------------------------------------------------------------------

def test_membership_boundaries(oracle_lib):
    means = np.array([[0.5, 0, 0], [0.5000001, 0, 0], [1, 1, 1], [2, 3, 4], [2, 3, 4.0001], [0, 0, 0]], np.float64)
    regions = [synth.Region(synth.REGION_SPHERE, np.zeros(3), np.zeros(3), 0.5),
               synth.Region(synth.REGION_AABB, np.array([1.0, 1, 1]), np.array([2.0, 3, 4]), 0.0)]
    sc = _scene(means, np.zeros((6, 3)), [[1, 0, 0, 0]] * 6, np.zeros(6), np.zeros((6, 1, 3)), 0, [_one_cam()],
                regions)
    sc.means = means
    assert list(oracle.membership(sc)) == [True, False, True, True, False, True]


def test_membership_brute_force_random(oracle_lib):
    sc = synth.make_scene("c3", n=20000, width=64, height=64, n_views=1, with_targets=False)
    act = oracle.membership(sc)
    m = sc.means.astype(np.float64)
    ref = np.zeros(sc.n, bool)
    for r in sc.regions:
        ref |= np.all((m >= r.a.astype(np.float64)) & (m <= r.b.astype(np.float64)), axis=1)
    assert np.array_equal(act, ref) and act.any()


# ---------------------------------------------------------------------------
# SH basis pins (R15): scipy's spherical harmonics and orthonormality
# ---------------------------------------------------------------------------

def test_sh_matches_scipy(oracle_lib):
    sp = pytest.importorskip("scipy.special")
    rng = np.random.default_rng(0)
    for _ in range(20):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        theta, phi = math.acos(d[2]), math.atan2(d[1], d[0])
        Y = oracle.sh_basis(3, d)
        for l in range(4):
            for m in range(-l, l + 1):
                c = sp.sph_harm_y(l, abs(m), theta, phi)
                std = math.sqrt(2) * (-1) ** m * (c.real if m > 0 else c.imag) if m != 0 else c.real
                # 3DGS basis = (-1)^m times the standard real SH (Condon-Shortley sign kept)
                assert Y[l * l + l + m] == pytest.approx((-1) ** m * std, abs=1e-12)


def test_sh_orthonormal(oracle_lib):
    # Gauss-Legendre in cos(theta) x uniform in phi: exact for polynomials of degree <= 6
    xs, ws = np.polynomial.legendre.leggauss(12)
    phis = np.linspace(0, 2 * np.pi, 24, endpoint=False)
    G = np.zeros((16, 16))
    for ct, wt in zip(xs, ws):
        st = math.sqrt(1 - ct * ct)
        for ph in phis:
            Y = oracle.sh_basis(3, [st * math.cos(ph), st * math.sin(ph), ct])
            G += wt * (2 * np.pi / len(phis)) * np.outer(Y, Y)
    assert np.allclose(G, np.eye(16), atol=1e-12)


# ---------------------------------------------------------------------------
# R5 near plane, R10 frustum clamp of J, R13 depth ties (previously unpinned)
# ---------------------------------------------------------------------------

def test_r5_near_plane_threshold(oracle_lib):
    """3DGS near plane (R5): culled iff t_z <= 0.2.  Camera R = I, t = 0, so t_z = z exactly
    (fp64 means)."""
    cam = _one_cam()
    zs = np.array([0.19, 0.2, 0.2 + 1e-12, 0.21, 0.5])
    means = np.stack([np.zeros(5), np.zeros(5), zs], 1)
    sc = _scene(means, np.log(np.full((5, 3), 0.002)), [[1, 0, 0, 0]] * 5, np.zeros(5), np.zeros((5, 1, 3)), 0,
                [cam])
    sc.means = means
    p = oracle.project(sc, 0)
    assert list(p["culled"]) == [1, 1, 0, 0, 0]
    assert p["tcam"][:, 2] == pytest.approx(zs, abs=0)


def _clamp_cam():
    # W = H = 64, f = 100: tan(fov_x / 2) = W / (2 f) = 0.32, clamp limit L = 1.3 * 0.32 = 0.416
    return _one_cam(W=64, H=64, f=100.0, cx=32.0, cy=32.0)


@pytest.mark.parametrize("xz,yz", [(0.5, 0.0), (-0.5, 0.0), (0.0, 0.47), (0.45, -0.46), (0.2, 0.1)])
def test_r10_frustum_clamp_closed_form(oracle_lib, xz, yz):
    """R10: J uses x/z, y/z clamped to +-1.3 tan(fov/2).  For an isotropic Gaussian (Sigma = s^2 I)
    seen by R = I the closed form is Sigma' = s^2 J J^T + 0.3 I with
    J = [[f/z, 0, -f xc/z], [0, f/z, -f yc/z]], xc = clamp(x/z, -L, L): A = (f s / z)^2 (1 + xc^2) + 0.3,
    B = (f s / z)^2 xc yc, C = (f s / z)^2 (1 + yc^2) + 0.3.  The centre u, v uses the UNclamped x/z."""
    L = 1.3 * 64 / (2 * 100.0)
    z, s = 2.0, 0.4                                   # a large splat: its footprint reaches the image
    means = np.array([[xz * z, yz * z, z]])
    sc = _scene(means, np.log([[s] * 3]), [[1, 0, 0, 0]], [0.0], np.zeros((1, 1, 3)), 0, [_clamp_cam()])
    sc.means = means
    sc.log_scales = np.log([[s] * 3])
    p = oracle.project(sc, 0)
    assert p["culled"][0] == 0
    xc, yc = min(max(xz, -L), L), min(max(yz, -L), L)
    k = (100.0 * s / z) ** 2
    assert p["cov2d"][0] == pytest.approx([k * (1 + xc * xc) + 0.3, k * xc * yc, k * (1 + yc * yc) + 0.3],
                                          rel=1e-12, abs=1e-9)
    assert p["uv"][0] == pytest.approx([100.0 * xz + 32.0 - 0.5, 100.0 * yz + 32.0 - 0.5], rel=1e-12)


def test_r13_depth_ties_by_index(oracle_lib):
    """R13: the depth key is the fp32 rounding of the fp64 view depth and equal keys are ordered by
    ascending Gaussian index -- even when the true (fp64) depths differ below fp32 resolution.
    Two coincident splats (opacity 0.5 red, 0.6 green): the transmittance product of V2 in index
    order, C = (0.5, 0.6 (1 - 0.5), 0) = (0.5, 0.3, 0); with the rows swapped, (0.5 (1 - 0.6), 0.6, 0)."""
    cam = _one_cam()
    for behind0 in (1e-9, 0.0):           # row 0 slightly BEHIND row 1 in fp64, same fp32 key; or exactly tied
        means = np.array([[0.0, 0.0, 2.0 + behind0], [0.0, 0.0, 2.0]])
        ops = np.log(np.array([0.5, 0.6]) / (1 - np.array([0.5, 0.6])))
        sh = _dc(np.array([[1.0, 0, 0], [0, 1.0, 0]])).reshape(2, 1, 3)
        for order in ((0, 1), (1, 0)):
            o = list(order)
            sc = _scene(means[o], np.log(np.full((2, 3), 0.05)), [[1, 0, 0, 0]] * 2, ops[o], sh[o], 0, [cam])
            sc.means, sc.opacity_logits, sc.sh = means[o], ops[o], sh[o]
            sc.log_scales = np.log(np.full((2, 3), 0.05))
            p = oracle.project(sc, 0)
            assert p["depth_key"][0] == p["depth_key"][1]
            r = oracle.render(sc, 0, np.ones(2, bool), p, use_target=False, with_grad=False)
            first_red = order == (0, 1)       # index 0 holds the red splat
            expect = [0.5, 0.3, 0.0] if first_red else [0.2, 0.6, 0.0]
            assert r["image"][:, 32, 32] == pytest.approx(expect, abs=1e-12)


def test_p7_finite_differences_clamped_jacobian(oracle_lib):
    """P7 on Gaussians whose J is frustum-clamped (R10) in x, in y and in both, next to an unclamped
    one: the clamped-branch derivative (dJ02/dt_x = 0, dJ02/dt_z = +-f L / t_z^2) against central
    finite differences of the smooth probe loss.  Every clamped Gaussian sits >= 0.05 beyond the limit
    and every unclamped one >= 0.05 inside it, so no +-1e-4 perturbation changes a clamp decision."""
    W = H = 32
    f = 40.0                                          # L = 1.3 * 32 / 80 = 0.52
    cam = synth.Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), f, f, 16.0, 16.0, W, H)
    L = 1.3 * W / (2 * f)
    z = np.array([3.0, 3.2, 3.4, 3.6])
    xz = np.array([0.60, 0.0, -0.62, 0.10])
    yz = np.array([0.0, 0.61, -0.60, 0.05])
    means = np.stack([xz * z, yz * z, z], 1)
    rng = np.random.default_rng(31)
    ls = np.log(rng.uniform(0.25, 0.4, (4, 3)))
    q = rng.standard_normal((4, 4))
    ops = np.log(np.array([0.5, 0.45, 0.55, 0.4]) / (1 - np.array([0.5, 0.45, 0.55, 0.4])))
    sh = rng.normal(0.0, 0.3, (4, 4, 3))
    sh[:, 0, :] = (rng.uniform(0.3, 0.7, (4, 3)) - 0.5) / C0
    sc = _f64_scene(_scene(means, ls, q, ops, sh, 1, [cam]))
    sc.means, sc.log_scales, sc.quats, sc.opacity_logits, sc.sh = means, ls, q, ops, sh
    p = oracle.project(sc, 0)
    assert np.all(p["culled"] == 0)
    tc = p["tcam"]
    rx, ry = np.abs(tc[:, 0] / tc[:, 2]), np.abs(tc[:, 1] / tc[:, 2])
    assert np.all(np.abs(rx - L) >= 0.05) and np.all(np.abs(ry - L) >= 0.05)
    assert (rx > L).sum() == 2 and (ry > L).sum() == 2      # x clamped twice, y clamped twice
    act = np.ones(4, bool)
    w = np.random.default_rng(32).standard_normal((1, 3, H, W))
    g = oracle.forward_backward(sc, active=act, dL_dC=w)["grad"]
    eps = 1e-4
    worst, checked = 0.0, 0
    for i in range(4):
        for name, count, col in (("means", 3, 0), ("quats", 4, 3), ("log_scales", 3, 7)):
            arr = getattr(sc, name)
            for j in range(count):
                x0 = arr[i, j]
                fds = []
                for h in (eps, eps / 2):
                    arr[i, j] = x0 + h
                    lp = _probe(sc, w, act)
                    arr[i, j] = x0 - h
                    lm = _probe(sc, w, act)
                    arr[i, j] = x0
                    assert _same_decisions(lp, lm)
                    fds.append((lp[0] - lm[0]) / (2 * h))
                fd = (4.0 * fds[1] - fds[0]) / 3.0
                an = g[i, col + j]
                err = abs(fd - an) / max(abs(fd), abs(an), 1e-8)
                worst = max(worst, err)
                checked += 1
                assert err < 1e-5, (name, i, j, fd, an)
    assert checked == 40


# ---------------------------------------------------------------------------
# decision replay of the parity protocol (test infrastructure)
# ---------------------------------------------------------------------------

def test_pixel_replay_baseline_equals_render(oracle_lib):
    """With no flip, the replay's per-pixel list (brute force over rects, (kappa, index) order)
    composites exactly what orc_render_view does: a 0 distance to the rendered image."""
    sc = synth.make_scene("c2", n=3000, width=96, height=80, n_views=1)
    fb = oracle.forward_backward(sc, with_grad=False)
    r = fb["renders"][0]
    ys, xs = np.nonzero(np.kron(r["tile_mask"], np.ones((16, 16), bool))[: sc.height, : sc.width])
    assert ys.size > 100
    for k in range(0, ys.size, 37):
        best, _ = oracle.pixel_replay(sc, 0, r["proj"], xs[k], ys[k], r["image"][:, ys[k], xs[k]])
        assert best == 0.0


def test_pixel_replay_skip_flip(oracle_lib):
    """V1's splat with its opacity tuned so that alpha = (1/255)(1 + 5e-6) at 8 px from the centre:
    the fp64 oracle composites it (C = c alpha), the pixel is flagged, and the replay explains a
    renderer that skipped it (C = 0) -- but not an arbitrary value."""
    cam = _one_cam()
    sig2 = (100.0 * 0.05 / 2.0) ** 2 + 0.3
    o = (1.0 / 255.0) * (1.0 + 5e-6) / math.exp(-0.5 * 64.0 / sig2)
    sc = _scene(np.array([[0.0, 0.0, 2.0]]), np.log([[0.05] * 3]), [[1, 0, 0, 0]], [math.log(o / (1 - o))],
                np.full((1, 1, 3), _dc(0.6)), 0, [cam])
    sc.means = np.array([[0.0, 0.0, 2.0]])
    sc.log_scales = np.log([[0.05] * 3])
    sc.opacity_logits = np.array([math.log(o / (1 - o))])
    p = oracle.project(sc, 0)
    r = oracle.render(sc, 0, np.ones(1, bool), p, use_target=False, with_grad=False)
    c = float(np.float32(_dc(0.6))) * C0 + 0.5
    assert r["image"][0, 32, 40] == pytest.approx(c / 255.0, rel=1e-4)
    assert r["ambiguous"][32, 40]
    best, nw = oracle.pixel_replay(sc, 0, p, 40, 32, np.zeros(3))
    assert nw >= 1 and best < 1e-12
    best, _ = oracle.pixel_replay(sc, 0, p, 40, 32, np.full(3, 0.001))
    assert best > 1e-4


def test_pixel_replay_termination_flip(oracle_lib):
    """Two coincident splats, alpha 0.99 then 0.989999: T' = 0.01 x 0.010001 = 1.0001e-4 >= 1e-4, so the
    oracle composites the second (R3); the window flags the test and the replay explains a renderer
    that terminated before it (C = 0.99 c1)."""
    sc = _coincident([0.995, 0.989999], [[1, 0, 0], [0, 1, 0]])
    r = oracle.render(sc, 0, np.ones(2, bool), use_target=False, with_grad=False)
    assert r["n_contrib"][32, 32] == 2
    assert r["ambiguous"][32, 32]
    p = oracle.project(sc, 0)
    best, nw = oracle.pixel_replay(sc, 0, p, 32, 32, np.array([0.99, 0.0, 0.0]))
    assert nw >= 1 and best < 1e-12


# ---------------------------------------------------------------------------
# NEXT-3 per-change-set activation: the oracle's per_set mode
# ---------------------------------------------------------------------------

def test_per_set_equals_independent_changes(oracle_lib):
    """"Apply our method in parallel to each change" (L397): with two change sets (one region and one
    view each), the per-set step's gradient is the SUM of the two single-change steps (each with its
    own regions and views, the same loss normalisation) and its loss is the sum of their losses; with
    every set id 0 it is the union step."""
    import dataclasses
    sc = synth.make_scene("c5", n=4000, width=96, height=64, n_views=10)
    sets = sorted({c.set for c in sc.cameras})
    assert len(sets) >= 2 and len({r.set for r in sc.regions}) >= 2
    V = len(sc.cameras)
    per = oracle.forward_backward(sc, per_set=True)
    tot = np.zeros_like(per["grad"])
    loss = 0.0
    for s in sets:
        views = [v for v in range(V) if sc.cameras[v].set == s]
        sub = dataclasses.replace(sc, regions=[r for r in sc.regions if r.set == s])
        fb = oracle.forward_backward(sub, views=views, n_views_total=V)
        tot += fb["grad"]
        loss += fb["loss"]
    assert np.allclose(per["grad"], tot, rtol=1e-12, atol=1e-300)
    assert per["loss"] == pytest.approx(loss, rel=1e-12)
    assert np.array_equal(per["idx"], oracle.forward_backward(sc, with_grad=False)["idx"])   # O^t = the union
    flat = dataclasses.replace(sc, cameras=[dataclasses.replace(c, set=0) for c in sc.cameras],
                               regions=[dataclasses.replace(r, set=0) for r in sc.regions])
    a, b = oracle.forward_backward(flat, per_set=True), oracle.forward_backward(sc)
    assert np.array_equal(a["grad"], b["grad"]) and a["loss"] == b["loss"]
