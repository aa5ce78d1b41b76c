"""Pins of the NEXT-2 oracle (oracle/voting.py) against values the paper's formulas fix by hand:
the voting inequality of PAPER.md L463 at its boundaries (the SPEC example N=25, c=12, o=0 is
excluded), centre projection on a hand-built camera (R11 pixel convention, behind-camera and
image-border cases, R34), and the sphere fit of L468-L469 on point sets with known mean and
distance quantiles (R35)."""
import numpy as np
import pytest

from oracle import voting as Vt
import synth


def _cam(W=64, H=64, f=100.0):
    return synth.Camera(np.eye(3, dtype=np.float32), np.zeros(3, np.float32), f, f, W / 2, H / 2, W, H)


def test_majority_boundaries():
    N = 25
    # c: N < 2c  <=>  c >= 13
    assert not Vt.majority(np.array([12]), np.array([0]), N)[0]    # 25 < 24 false (SPEC example)
    assert Vt.majority(np.array([13]), np.array([0]), N)[0]
    # o: (4/3) o < N  <=>  4 o < 75  <=>  o <= 18
    assert Vt.majority(np.array([25]), np.array([18]), N)[0]
    assert not Vt.majority(np.array([25]), np.array([19]), N)[0]
    # N = 3: o = 2 -> 8 < 9 true; c = 2 -> 3 < 4 true
    assert Vt.majority(np.array([2]), np.array([2]), 3)[0]


def test_vote_counts_hand_camera():
    cam = _cam(f=128.0)                       # u = 128 x / z + 32: exact in fp32 / fp64 for the values below
    mask = np.zeros((1, 64, 64), np.uint8)
    mask[0, 32, 32] = 1
    means = np.array([[0.0, 0.0, 2.0],        # u = w = 32 -> pixel (32, 32): in the mask
                      [0.015625, 0.0, 2.0],   # u = 33 -> pixel 33: in the image, not in the mask
                      [0.0, 0.0, -1.0],       # behind the camera: outside
                      [0.5, 0.0, 2.0],        # u = 64.0 exactly: outside [0, 64)
                      [0.49609375, 0.0, 2.0], # u = 63.75: pixel 63, inside
                      [-0.5, 0.0, 2.0]],      # u = 0.0: inside (pixel 0)
                     np.float32)
    c, o = Vt.vote_counts(means, [cam], mask)
    assert c.tolist() == [1, 0, 0, 0, 0, 0]
    assert o.tolist() == [0, 0, 1, 1, 0, 0]


def test_fit_spheres_known_quantiles():
    rng = np.random.default_rng(0)
    centre = np.array([1.0, -2.0, 0.5])
    # cluster 0: 100 points on the unit sphere in antipodal pairs (mean exactly the centre), all d = 1
    d = rng.standard_normal((50, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    p0 = np.concatenate([centre + d, centre - d])
    # cluster 1: antipodal pairs at distances 1..50 along x (100 points, mean = origin)
    dist = np.arange(1, 51, dtype=np.float64)
    p1 = np.concatenate([np.stack([dist, 0 * dist, 0 * dist], 1), np.stack([-dist, 0 * dist, 0 * dist], 1)])
    pts = np.concatenate([p0, p1, [[9.0, 9.0, 9.0]]])
    labels = np.array([0] * 100 + [1] * 100 + [-1])     # the last point is noise
    c, r = Vt.fit_spheres(pts, labels, 2)
    assert np.allclose(c[0], centre, atol=1e-12) and np.allclose(c[1], 0.0, atol=1e-12)
    assert r[0] == pytest.approx(1.1, rel=1e-12)
    # sorted distances 1,1,2,2,...,50,50: h = 99 * 0.98 = 97.02 -> d[97] = 49, d[98] = 50 -> 49.02
    assert r[1] == pytest.approx(1.1 * 49.02, rel=1e-12)
