"""CPU ORACLE for the NEXT-3/NEXT-4 rows: history record/recover and the merge of
batched updates (TEST INFRASTRUCTURE -- only tests/ may import this module; the product package
never does and shares no code with it).

Plain numpy, step by step from PAPER.md:
* record -- Supp. "History Recovery" (L656-L672): "we store O^t and I^t immediately after computing
  O^t, before any optimization"; I^t is the indicator of O^t over the rows of G^{t-1}; "before
  optimization, we rearrange the Gaussian order to ensure G^t[:#static] = G^{t-1}_static".
* recover -- Algorithm "History Recovery" (L684-L701): N = G^T[:|not I^T|] + O^T (array of the
  target size); N[I^T] = O^T; N[not I^T] = the static prefix, both in order; repeated per step.
* merge -- Supp. "Batched Updates" (L642-L648): G^t = O^t_1 u O^t_2 u G^{t-1}[not I_1 and not I_2].
  The printed equation reads "G^{t-1} minus G^{t-1}[not I_1 and not I_2]", which would drop exactly
  the unchanged Gaussians the sentence says are retained; reading R36 keeps the
  unchanged Gaussians: [unchanged rows in order][O_1][O_2].
Rows are any per-Gaussian arrays (dict of equal-length arrays).
"""
from __future__ import annotations

import numpy as np


def record(params: dict, I: np.ndarray):
    """(O^t rows in order, I^t as uint8) -- the stored history of one step."""
    I = np.asarray(I, bool)
    return {k: np.asarray(v)[I].copy() for k, v in params.items()}, I.astype(np.uint8)


def recover_one(params_t: dict, O: dict, I: np.ndarray) -> dict:
    """G^{t-1} from G^t (whose first |not I| rows are the static rows of G^{t-1}), O^t and I^t."""
    I = np.asarray(I, bool)
    n_static = int((~I).sum())
    out = {}
    for k, v in params_t.items():
        v = np.asarray(v)
        N = np.empty((len(I),) + v.shape[1:], v.dtype)
        N[I] = np.asarray(O[k])
        N[~I] = v[:n_static]
        out[k] = N
    return out


def recover(params_T: dict, history, n_back: int) -> dict:
    """RecoverState: apply recover_one for the last `n_back` stored steps, newest first.
    history = [(O^t, I^t) for t = 1..T] in time order."""
    cur = params_T
    for O, I in reversed(history[len(history) - n_back:]):
        cur = recover_one(cur, O, I)
    return cur


def merge(params_prev: dict, O1: dict, I1: np.ndarray, O2: dict, I2: np.ndarray) -> dict:
    """Batched updates (reading R36): [G^{t-1}[not I1 and not I2]][O1][O2]."""
    keep = ~np.asarray(I1, bool) & ~np.asarray(I2, bool)
    return {k: np.concatenate([np.asarray(v)[keep], np.asarray(O1[k]), np.asarray(O2[k])])
            for k, v in params_prev.items()}
