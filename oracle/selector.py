"""Importance-weighted mini-batch selection restated (TEST INFRASTRUCTURE).

Follows selector.py:36-61 of the reference:

  init_scores(n, gamma)         scores = 0.5 + gamma            (:36-43)
  select_batch(scores, b, rng)  p = scores / scores.sum();
                                rng.choice(n, b, replace=False, p=p);
                                sorted + base_eid               (:46-53)
  update_scores(...)            scores[eids - base] = sigmoid(logits) + gamma,
                                IndexError outside the range    (:56-61)

numpy's Generator.choice(replace=False, p=...) is restated step by step
(``choice_wor``) because the device kernel (select.cu) reproduces exactly
this sequence: rounds of ``random(size - n_uniq)`` draws, found entries
zeroed in p, sequential ``cumsum``, normalisation by the last element,
``searchsorted(side='right')``, first-occurrence de-duplication.  The
restatement is pinned against numpy itself (tests/test_oracle_golden.py)
and against the reference's select_batch (golden ``selector.npz``).
"""

from __future__ import annotations

import numpy as np


def pairwise_sum(a):
    """numpy's float64 add.reduce order (loops_utils.h pairwise_sum): blocks
    of <= 128 with 8 strided accumulators, halves split at a multiple of 8."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    if n < 8:
        res = 0.0
        for v in a:
            res += v
        return float(res)
    if n <= 128:
        r = a[:8].copy()
        i = 8
        while i < n - (n % 8):
            r += a[i:i + 8]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[i]
            i += 1
        return float(res)
    n2 = n // 2
    n2 -= n2 % 8
    return float(pairwise_sum(a[:n2]) + pairwise_sum(a[n2:]))


def choice_wor(rng, n, size, p):
    """Generator.choice(n, size, replace=False, p=p) restated."""
    p = np.array(p, dtype=np.float64, copy=True)
    if np.count_nonzero(p > 0) < size:
        raise ValueError("Fewer non-zero entries in p than size")
    found = np.zeros(size, dtype=np.int64)
    n_uniq = 0
    while n_uniq < size:
        x = rng.random(size - n_uniq)
        if n_uniq > 0:
            p[found[:n_uniq]] = 0
        cdf = np.cumsum(p)
        cdf /= cdf[-1]
        new = cdf.searchsorted(x, side="right")
        _, first = np.unique(new, return_index=True)
        first.sort()
        new = new.take(first)
        found[n_uniq:n_uniq + new.size] = new
        n_uniq += new.size
    return found


def init_scores(num_train_edges, gamma=0.1):
    if num_train_edges < 1:
        raise ValueError("need at least one training edge")
    if gamma < 0:
        raise ValueError("gamma must be >= 0")
    return np.full(num_train_edges, 0.5 + gamma)


def select_batch(scores, b, rng, base_eid=0):
    scores = np.asarray(scores, dtype=np.float64)
    if b > scores.shape[0]:
        raise ValueError(f"batch size {b} exceeds {scores.shape[0]} training edges")
    p = scores / pairwise_sum(scores)
    return np.sort(choice_wor(rng, scores.shape[0], b, p)) + base_eid


def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    e = np.exp(-np.abs(x))
    return np.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def update_scores(scores, batch_eids, logits, gamma, base_eid=0):
    idx = np.asarray(batch_eids, dtype=np.int64) - base_eid
    if idx.size and (idx.min() < 0 or idx.max() >= scores.shape[0]):
        raise IndexError("eid outside the training range")
    scores[idx] = sigmoid(logits) + gamma
    return scores


# ---- golden cases (tests/golden/make_golden.py selector_cases) --------------
SELECTOR_CASES = [("init", 5000, 600, 11), ("random", 20000, 600, 12), ("few", 60, 50, 13), ("zeros", 3000, 200, 14),
                  ("short", 40000, 600, 15), ("skewed", 7001, 300, 16), ("random", 1_000_003, 600, 17),
                  ("short", 2_000_000, 1000, 18), ("skewed", 500_000, 4000, 19)]


def case_scores(kind, n, seed):
    """Deterministic score vectors of the selector golden cases."""
    r = np.random.default_rng(seed)
    if kind == "init":
        return np.full(n, 0.6)
    if kind == "random":
        return 1.0 / (1.0 + np.exp(-r.normal(size=n) * 3)) + 0.1
    if kind == "zeros":
        s = r.random(n) + 0.05
        s[r.random(n) < 0.5] = 0.0
        return s
    if kind == "short":  # few significant bits: exact sums and rounding ties in the cumsum
        return r.integers(1, 5, n).astype(np.float64)
    if kind == "skewed":
        return r.random(n) ** 8 + 1e-9
    raise ValueError(kind)


def pcg_generator(words):
    """numpy Generator at the PCG64 (state, inc) stored as 4 uint64 words."""
    w = [int(x) for x in words]
    bg = np.random.PCG64()
    bg.state = {"bit_generator": "PCG64", "state": {"state": (w[0] << 64) | w[1], "inc": (w[2] << 64) | w[3]},
                "has_uint32": 0, "uinteger": 0}
    return np.random.Generator(bg)
