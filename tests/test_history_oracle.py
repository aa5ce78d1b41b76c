"""Pins of the NEXT-3/4 oracle (oracle/history.py) against the paper's statements, by construction
independent of its code: recovery is exact ("identical reconstructions to storing the
full scene"), multi-step recovery walks back any number of steps, the static prefix invariant of
L666, and the batched-update merge keeps every unchanged Gaussian (L645, reading R36)."""
import numpy as np

from oracle import densify as D
from oracle import history as Hs


def _scene(n, rng):
    return {"means": rng.standard_normal((n, 3)), "opacity_logits": rng.standard_normal(n),
            "sh": rng.standard_normal((n, 4, 3))}


def _step(params, rng, frac=0.2):
    """One timestep as the method runs it: O^t chosen, history recorded, partition (static prefix),
    O^t optimised (changed values, pruned and densified rows -- only the suffix changes)."""
    n = len(params["means"])
    I = rng.random(n) < frac
    O, Ib = Hs.record(params, I)
    perm, ns = D.partition_static(I)
    new = {k: np.asarray(v)[perm].copy() for k, v in params.items()}
    # optimisation touches only the suffix: perturb, drop one row, append two
    m = len(new["means"])
    keep = np.ones(m, bool)
    if m > ns:
        keep[ns + rng.integers(0, m - ns)] = False
    for k in new:
        v = new[k][keep]
        v[ns:] = v[ns:] + 0.5
        extra = rng.standard_normal((2,) + v.shape[1:])
        new[k] = np.concatenate([v, extra])
    return new, (O, Ib), ns


def test_recover_is_exact_over_several_steps():
    rng = np.random.default_rng(0)
    states = [_scene(200, rng)]
    history = []
    for t in range(4):
        nxt, h, ns = _step(states[-1], rng)
        # static prefix invariant: G^t[:#static] = G^{t-1}_static, in order
        for k in nxt:
            assert np.array_equal(nxt[k][:ns], np.asarray(states[-1][k])[h[1] == 0])
        states.append(nxt)
        history.append(h)
    for back in range(1, 5):
        rec = Hs.recover(states[-1], history, back)
        for k in states[0]:
            assert np.array_equal(rec[k], states[-1 - back][k]), (back, k)


def test_history_storage_is_the_changed_rows_only():
    rng = np.random.default_rng(1)
    g = _scene(1000, rng)
    I = np.zeros(1000, bool)
    I[::20] = True
    O, Ib = Hs.record(g, I)
    assert len(O["means"]) == 50 and Ib.sum() == 50 and len(Ib) == 1000


def test_merge_keeps_unchanged_and_both_updates():
    rng = np.random.default_rng(2)
    g = _scene(10, rng)
    I1 = np.zeros(10, bool); I1[[1, 2]] = True
    I2 = np.zeros(10, bool); I2[[2, 7]] = True
    O1 = _scene(3, rng)
    O2 = _scene(1, rng)
    out = Hs.merge(g, O1, I1, O2, I2)
    unchanged = [0, 3, 4, 5, 6, 8, 9]
    assert len(out["means"]) == 7 + 3 + 1
    assert np.array_equal(out["means"][:7], g["means"][unchanged])
    assert np.array_equal(out["means"][7:10], O1["means"]) and np.array_equal(out["means"][10:], O2["means"])
