"""Edge-feature cache restated (TEST INFRASTRUCTURE).  Follows cache.py:58-136.

k / epsilon rules (cache.py:58-69), per-occurrence counting and hit/miss
stats (:72-86), top-k of touched edges by (count desc, eid asc) (:89-104),
replace iff overlap < epsilon, counters reset either way (:107-118), and the
clairvoyant per-epoch oracle (:121-136).
"""

from __future__ import annotations

import numpy as np


class OracleCache:
    def __init__(self, num_edges, k, epsilon=None, features=None):
        if 0 < k < 1:
            k = int(k * num_edges)
        k = int(k)
        if epsilon is None:
            epsilon = 0.9
        if isinstance(epsilon, float) and 0 < epsilon <= 1:
            epsilon = int(np.ceil(epsilon * k))
        self.num_edges, self.k, self.epsilon = int(num_edges), k, int(epsilon)
        self.features = features
        self.resident = np.zeros(self.num_edges, dtype=bool)
        self.counters = np.zeros(self.num_edges, dtype=np.int64)
        self.epochs = [[0, 0]]          # [hits, misses] per epoch
        self.replacements = []

    def lookup(self, eids):
        eids = np.asarray(eids, dtype=np.int64).ravel()
        if eids.size and (eids.min() < 0 or eids.max() >= self.num_edges):
            raise IndexError(f"edge id out of range [0, {self.num_edges})")
        hits = self.resident[eids]
        self.counters += np.bincount(eids, minlength=self.num_edges)
        h = int(hits.sum())
        self.epochs[-1][0] += h
        self.epochs[-1][1] += int(eids.size) - h
        feats = None if self.features is None else self.features[eids]
        return feats, hits

    def maybe_replace(self):
        top = topk_edges(self.counters, self.k)
        overlap = int(self.resident[top].sum())
        replaced = overlap < self.epsilon
        if replaced:
            self.resident[:] = False
            self.resident[top] = True
        self.replacements.append(bool(replaced))
        self.counters[:] = 0
        self.epochs.append([0, 0])
        return replaced


def topk_edges(counts, k):
    """Touched edges, k largest by (count desc, eid asc) (cache.py:89-104)."""
    counts = np.asarray(counts)
    touched = np.flatnonzero(counts)
    if touched.size == 0 or k == 0:
        return np.empty(0, dtype=np.int64)
    order = np.lexsort((touched, -counts[touched]))    # count desc, then eid asc
    return touched[order[:k]]


def oracle_rates(trace_counts, k):
    rates = []
    for epoch in np.asarray(trace_counts):
        total = int(epoch.sum())
        if total == 0:
            rates.append(None)
            continue
        rates.append(float(epoch[topk_edges(epoch, k)].sum() / total))
    return rates
