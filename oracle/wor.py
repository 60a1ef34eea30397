"""Policy sampling without replacement restated (TEST INFRASTRUCTURE).

Follows sampler.py:138-176: n rounds over the batch; per round the row
total (numpy pairwise sum), alive = total > 1e-12, u = rng.random(B) *
total, pick = min(#(cumsum < u), m-1), zero the pick; then a stable
ascending sort of the picks and log q gathered at the picks times the mask.
"""

from __future__ import annotations

import numpy as np


def sample_wor(q, log_q, n, rng, B_global=None, global_rows=None):
    """global_rows/B_global: this shard's rows inside the full batch; round
    k's draw for global row g is stream output k*B_global + g (sampler.py:154)."""
    probs = np.array(q, dtype=np.float64)
    B, m = probs.shape
    if B_global is None:
        B_global, global_rows = B, np.arange(B)
    sel = np.full((B, n), -1, dtype=np.int64)
    smask = np.zeros((B, n), dtype=bool)
    rows = np.arange(B)
    for k in range(n):
        total = probs.sum(axis=1)
        live = total > 1e-12
        if not live.any():
            break
        u = rng.random(B_global)[global_rows] * total
        below = (np.cumsum(probs, axis=1) < u[:, None]).sum(axis=1)
        pick = np.minimum(below, m - 1)
        sel[live, k] = pick[live]
        smask[live, k] = True
        probs[rows[live], pick[live]] = 0.0
    key = np.where(smask, sel, np.iinfo(np.int64).max)
    order = np.argsort(key, axis=1, kind="stable")
    sel = np.take_along_axis(sel, order, axis=1)
    smask = np.take_along_axis(smask, order, axis=1)
    slq = None
    if log_q is not None:
        lq = np.asarray(log_q)
        slq = lq[rows[:, None], np.maximum(sel, 0)] * smask.astype(lq.dtype)
    return sel, smask, slq
