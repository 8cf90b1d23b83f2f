"""fp64 oracle of the ring-attention LSE merge.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Two partial attention results over disjoint key sets K1, K2 of the same query
rows, (O1, LSE1) and (O2, LSE2), combine into the result over K1 u K2 by the
same rescale-and-add the paper's forward applies between key tiles (the running
max moves and O is multiplied by exp2(m_old - m_new) before the new block is
added: P:1398-1400), written with logsumexps instead of (max, sum) pairs:

    LSE = ln(exp(LSE1) + exp(LSE2))
    O   = exp(LSE1 - LSE) O1 + exp(LSE2 - LSE) O2

A row with LSE1 = LSE2 = -inf (no key in either set) stays O = 0, LSE = -inf
(reading #22). Layouts: O [..., N, H, d], LSE [..., H, N] (dense attention's).
"""
from __future__ import annotations

import numpy as np


def attn_merge(O1, LSE1, O2, LSE2):
    O1 = np.asarray(O1, dtype=np.float64)
    O2 = np.asarray(O2, dtype=np.float64)
    L1 = np.asarray(LSE1, dtype=np.float64)
    L2 = np.asarray(LSE2, dtype=np.float64)
    m = np.maximum(L1, L2)
    dead = np.isneginf(m)
    m0 = np.where(dead, 0.0, m)
    e1, e2 = np.exp(L1 - m0), np.exp(L2 - m0)
    s = e1 + e2
    with np.errstate(divide="ignore", invalid="ignore"):
        L = np.where(dead, -np.inf, m0 + np.log(s))
        w1 = np.where(dead, 0.0, e1 / s)
        w2 = np.where(dead, 0.0, e2 / s)
    # weights are [..., H, N]; O is [..., N, H, d]
    w1o = np.swapaxes(w1, -1, -2)[..., None]
    w2o = np.swapaxes(w2, -1, -2)[..., None]
    return w1o * O1 + w2o * O2, L
