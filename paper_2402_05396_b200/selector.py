"""Importance-weighted training-edge selection on the device (K9).

Drop-in for selector.py of the reference: the same
``ImportanceScores`` / ``init_scores`` / ``select_batch`` / ``update_scores``
API (selector.py:27-61) with the scores held in HBM.  ``select_batch``
reproduces ``rng.choice(n, b, replace=False, p=scores/scores.sum())``
bit for bit from the generator's PCG64 state (select.cu) and advances the
caller's generator by the draws it consumed, so a Trainer that keeps using
the stream sees the reference's state.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr, to_device
from .seeds import pcg_state


class IndexError_(IndexError):
    """Edge id outside the training range (selector.py:16-17)."""


@dataclass
class ImportanceScores:
    scores: object          # f64 CUDA tensor [num_train_edges]
    gamma: float
    base_eid: int = 0       # eid of the first training edge

    @property
    def num_edges(self):
        return int(self.scores.shape[0])


def init_scores(num_train_edges, gamma=0.1, base_eid=0):
    """Uniform start at sigmoid(0) + gamma (selector.py:36-43)."""
    if num_train_edges < 1:
        raise ValueError("need at least one training edge")
    if gamma < 0:
        raise ValueError("gamma must be >= 0")
    t = _lib.torch()
    _lib.require_cuda("init_scores")
    s = t.full((int(num_train_edges),), 0.5 + gamma, dtype=t.float64, device="cuda")
    return ImportanceScores(s, float(gamma), int(base_eid))


def as_scores(scores, gamma, base_eid=0):
    """Wrap an existing score vector (numpy or tensor) as device scores."""
    t = _lib.torch()
    return ImportanceScores(to_device(scores, t.float64), float(gamma), int(base_eid))


def select_batch(scores, b, rng):
    """b distinct training eids, probability proportional to the scores,
    sorted ascending (selector.py:46-53); int64 CUDA tensor."""
    t = _lib.torch()
    if b > scores.num_edges:
        raise ValueError(f"batch size {b} exceeds {scores.num_edges} training edges")
    state, inc = pcg_state(rng)
    p = _lib.tg_pcg64()
    p.state_hi, p.state_lo = _lib.u128_split(state)
    p.inc_hi, p.inc_lo = _lib.u128_split(inc)
    out = t.empty(int(b), dtype=t.int64, device=scores.scores.device)
    draws = _lib.c_int64(0)
    check(_lib.lib.tg_select_batch(ptr(scores.scores), scores.num_edges, int(b), p, int(scores.base_eid), ptr(out),
                                   _lib.ctypes.byref(draws), stream_ptr()))
    bg = rng.bit_generator if hasattr(rng, "bit_generator") else rng
    bg.advance(int(draws.value))  # the reference's choice() consumed these doubles
    return out


def _sigmoid(x):
    """selector.py's numerically stable logistic, in numpy (host logits)."""
    import numpy as np
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def update_scores(scores, batch_eids, logits):
    """Overwrite scores of positive batch edges with sigmoid(logit) + gamma
    (selector.py:56-61, Eq. 10).  The reference hands over host logits
    (``pos_logits.data``, training.py:403-404): those are mapped through the
    reference's own numpy expression -- 600 values, so the updated scores are
    bit-identical to the reference's -- and scattered on the device.  CUDA
    logits are mapped on the device (exp within 1 ulp of numpy's).  A
    repeated eid takes the value of its last position, like numpy."""
    t = _lib.torch()
    e = to_device(batch_eids, t.int64).reshape(-1)
    host = not isinstance(logits, t.Tensor)
    if host:
        vals = to_device(_sigmoid(logits).reshape(-1) + scores.gamma, t.float64)
    else:
        vals = to_device(logits, t.float64).reshape(-1)
    if vals.shape[0] != e.shape[0]:
        raise ValueError("one logit per batch edge")
    try:
        if host:
            check(_lib.lib.tg_scatter_scores(ptr(scores.scores), scores.num_edges, ptr(e), int(e.shape[0]),
                                             int(scores.base_eid), ptr(vals), stream_ptr()))
        else:
            check(_lib.lib.tg_update_scores(ptr(scores.scores), scores.num_edges, ptr(e), int(e.shape[0]),
                                            int(scores.base_eid), ptr(vals), float(scores.gamma), stream_ptr()))
    except IndexError as exc:
        raise IndexError_(str(exc)) from None
    return scores
