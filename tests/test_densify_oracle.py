"""Pins of the NEXT-1 oracle (oracle/densify.py) against what the paper and 3DGS fix, independent
of the oracle's own code: the static-prefix invariant, pruning only O^t
(L509-L511, L670), the split arithmetic (SPEC "densify_and_prune" example: one large high-gradient
Gaussian -> 2 children with scale / 1.6, scene size +1) and the clone rule."""
import math

import numpy as np
import pytest

from oracle import densify as D
import synth


def _sphere(c, r):
    return synth.Region(synth.REGION_SPHERE, np.asarray(c, np.float32), np.zeros(3, np.float32), float(r))


def test_partition_static_prefix_invariant():
    rng = np.random.default_rng(0)
    active = rng.random(50) < 0.3
    perm, ns = D.partition_static(active)
    assert ns == int((~active).sum())
    # G^t[:#static] = G_static^{t-1} in order, then O^t in order
    assert np.array_equal(perm[:ns], np.nonzero(~active)[0])
    assert np.array_equal(perm[ns:], np.nonzero(active)[0])
    assert sorted(perm.tolist()) == list(range(50))


def test_inside_regions_inclusive_boundary():
    m = np.array([[1.0, 0, 0], [1.0000001, 0, 0], [0, 0, 0]], np.float32)
    ins = D.inside_regions(m, [_sphere([0, 0, 0], 1.0)])
    assert ins.tolist() == [True, False, True]
    box = synth.Region(synth.REGION_AABB, np.array([0, 0, 0], np.float32), np.array([1, 1, 1], np.float32), 0.0)
    assert D.inside_regions(np.array([[1, 1, 1], [1, 1, 1.5]], np.float32), [box]).tolist() == [True, False]


def test_prune_only_suffix_and_keeps_order():
    # rows 0..2 static (two of them far outside the sphere: static Gaussians are never pruned),
    # rows 3..7 O^t: rows 4 and 6 have left the sphere
    means = np.array([[9, 9, 9], [0, 0, 0], [-9, 0, 0],
                      [0.1, 0, 0], [2, 0, 0], [0, 0.2, 0], [0, 0, -3], [0, 0, 0.9]], np.float32)
    keep = D.prune_outside(means, 3, [_sphere([0, 0, 0], 1.0)])
    assert keep.tolist() == [0, 1, 2, 3, 5, 7]


def _params(n, K=1):
    rng = np.random.default_rng(1)
    q = rng.standard_normal((n, 4))
    return {"means": rng.standard_normal((n, 3)), "log_scales": rng.uniform(-5, -2, (n, 3)),
            "quats": q / np.linalg.norm(q, axis=1, keepdims=True), "opacity_logits": rng.standard_normal(n),
            "sh": rng.standard_normal((n, K, 3)), "m_all": rng.standard_normal((n, 4)),
            "v_all": rng.random((n, 4))}


def test_split_arithmetic_identity_rotation():
    p = _params(3)
    p["quats"][2] = [1.0, 0, 0, 0]
    p["log_scales"][2] = np.log([0.1, 0.05, 0.02])
    accum = np.array([0, 0, 1e-3 * 4], np.float64)
    count = np.array([0, 0, 4])
    normals = np.zeros((3, 2, 3))
    normals[2, 0] = [1.0, -2.0, 0.5]
    normals[2, 1] = [0.0, 1.0, 3.0]
    out, kind = D.densify(p, 1, accum, count, normals, 2e-4, math.log(0.05))
    assert kind.tolist() == [0, 0, 2]
    assert len(out["means"]) == 4                                   # scene size +1
    mu = p["means"][2]
    assert np.allclose(out["means"][2], mu + np.array([0.1, -0.1, 0.01]), atol=1e-12)   # child 0: mu + s*z
    assert np.allclose(out["means"][3], mu + np.array([0.0, 0.05, 0.06]), atol=1e-12)   # child 1
    assert np.allclose(out["log_scales"][2:], np.log([0.1, 0.05, 0.02]) - np.log(1.6), atol=1e-12)  # scale / 1.6
    assert np.array_equal(out["opacity_logits"][2:], [p["opacity_logits"][2]] * 2)
    assert not out["m_all"][2:].any() and not out["v_all"][2:].any()  # fresh Adam state
    assert np.array_equal(out["means"][:2], p["means"][:2])        # the rest untouched


def test_split_rotation_quarter_turn():
    p = _params(1)
    c = math.cos(math.pi / 4)
    p["quats"][0] = [c, 0, 0, c]            # 90 degrees about z: x -> y
    p["log_scales"][0] = np.log([0.2, 0.1, 0.1])
    normals = np.zeros((1, 2, 3))
    normals[0, 0] = [1.0, 0, 0]
    out, kind = D.densify(p, 0, np.array([1.0]), np.array([1]), normals, 2e-4, math.log(0.05))
    assert kind.tolist() == [2]
    assert np.allclose(out["means"][0], p["means"][0] + np.array([0.0, 0.2, 0.0]), atol=1e-12)


def test_clone_small_and_threshold():
    p = _params(4)
    p["log_scales"][:] = np.log(0.01)
    accum = np.array([1.0, 1e-4, 3e-4, 5e-4])
    count = np.array([1, 1, 1, 0])          # row 3: never visible -> gradient 0
    out, kind = D.densify(p, 1, accum, count, np.zeros((4, 2, 3)), 2e-4, math.log(0.05))
    # row 0 is static (prefix) even with a large gradient; row 1 below the threshold; row 2 cloned
    assert kind.tolist() == [0, 0, 1, 0]
    assert len(out["means"]) == 5
    assert np.array_equal(out["means"][4], p["means"][2]) and np.array_equal(out["sh"][4], p["sh"][2])
    assert not out["m_all"][4].any() and np.array_equal(out["m_all"][:4], p["m_all"])


def test_below_threshold_unchanged():
    p = _params(5)
    out, kind = D.densify(p, 0, np.full(5, 1e-5), np.ones(5, np.int64), np.zeros((5, 2, 3)), 2e-4, -3.0)
    assert not kind.any()
    for k in p:
        assert np.array_equal(out[k], p[k])


def test_densify_stats_ndc_scaling():
    acc, cnt = D.densify_stats(np.zeros(3), np.zeros(3, np.int64), np.array([2]),
                               np.array([[[3e-6, -4e-6]], [[1e-6, 0.0]]]), np.array([[True], [False]]),
                               width=200, height=100, n_views_total=2)
    # || (3e-6 * 100 * 2, -4e-6 * 50 * 2) || = || (6e-4, -4e-4) ||; the invisible view does not count
    assert cnt.tolist() == [0, 0, 1]
    assert acc[2] == pytest.approx(math.hypot(6e-4, 4e-4), rel=1e-12)
