"""HBM edge-feature cache with top-k frequency replacement (K5 + K6).

Drop-in for cache.py of the reference: ``make_cache`` (:58), ``lookup``
(:72), ``maybe_replace`` (:107), ``oracle_cache`` (:121), ``run_trace``
(:139), ``cache_report`` (:150) with the same semantics, and a
``CacheState`` whose state lives on the device:

  slot_of  int32[E]   >= 0 iff the edge is resident (reference ``resident``);
                      the value is the row of the hot tier when one exists
  counters int32[E]   per-epoch access counts (reference ``counters``)
  stats    uint64[2]  hits / misses of the open epoch

Feature values never depend on residency (cache.py:85).  With ``hot_tier``
the resident rows are additionally copied into a dense [k, d] HBM block and
served from it; that is the placement used when the full table does not
live in local HBM (sharded / host tiers), and it changes no result.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr, to_device
from .graph import as_padded_table, feat_store, padded_rows


class EpochStats:
    """hits/misses of one epoch.  The open epoch reads the device counters."""

    def __init__(self, state=None, hits=0, misses=0):
        self._state = state
        self._hits, self._misses = int(hits), int(misses)

    def _sync(self):
        if self._state is not None:
            h = self._state.stats.cpu().numpy()
            return int(h[0]) + self._hits, int(h[1]) + self._misses
        return self._hits, self._misses

    @property
    def hits(self):
        return self._sync()[0]

    @property
    def misses(self):
        return self._sync()[1]

    @property
    def requests(self):
        h, m = self._sync()
        return h + m

    def hit_rate(self):
        h, m = self._sync()
        return h / (h + m) if (h + m) else None

    def close(self):
        self._hits, self._misses = self._sync()
        self._state = None


@dataclass
class CacheState:
    num_edges: int
    k: int
    epsilon: int
    features: object = None
    slot_of: object = None
    counters_i32: object = None
    stats: object = None
    hot: object = None
    epoch_stats: list = field(default_factory=list)
    replacements: list = field(default_factory=list)
    sim_fast_cost: float = 0.0
    sim_slow_cost: float = 0.0

    def __post_init__(self):
        t = _lib.torch()
        _lib.require_cuda("the feature cache")
        dev = t.device("cuda", t.cuda.current_device())
        if self.slot_of is None:
            self.slot_of = t.full((self.num_edges,), -1, dtype=t.int32, device=dev)
        if self.counters_i32 is None:
            self.counters_i32 = t.zeros(self.num_edges, dtype=t.int32, device=dev)
        if self.stats is None:
            self.stats = t.zeros(2, dtype=t.int64, device=dev)
        if not self.epoch_stats:
            self.epoch_stats.append(EpochStats(self))

    # reference-typed views -------------------------------------------------
    @property
    def resident(self):
        return self.slot_of >= 0

    @property
    def counters(self):
        return self.counters_i32.to(_lib.torch().int64)

    @property
    def resident_count(self):
        return int((self.slot_of >= 0).sum().item())

    def c_cache(self):
        return _lib.tg_cache_dev(ptr(self.slot_of), ptr(self.counters_i32), ptr(self.stats), int(self.num_edges))

    def c_store(self):
        if self.features is None:
            return None
        if self.hot is not None:
            return feat_store(self.features, self.hot, int(self.hot.stride(0)))
        return feat_store(self.features)


def make_cache(num_edges, k, epsilon=None, features=None, hot_tier=False):
    """k and epsilon may be absolute counts or fractions (of num_edges and of
    k respectively); epsilon defaults to 0.9 * k (cache.py:58-69)."""
    if 0 < k < 1:
        k = int(k * num_edges)
    k = int(k)
    if epsilon is None:
        epsilon = 0.9
    if 0 < epsilon <= 1 and isinstance(epsilon, float):
        epsilon = int(np.ceil(epsilon * k))
    t = _lib.torch()
    if features is not None and not hasattr(features, "c_store"):  # dense table (else placement.ShardedTable)
        features = as_padded_table(to_device(features, t.float32, rows_ok=True))
    state = CacheState(num_edges=int(num_edges), k=k, epsilon=int(epsilon), features=features)
    if hot_tier and features is not None and k > 0:
        state.hot = padded_rows((k,), int(features.shape[1]), features.device)
    return state


def lookup(state, eids, slow_cost_per_row=0.0):
    """Serve features for ``eids`` (either tier), count each occurrence, and
    return per-eid hit flags (cache.py:72-86)."""
    t = _lib.torch()
    host = not isinstance(eids, t.Tensor)
    e = to_device(eids, t.int64).reshape(-1)
    n = int(e.shape[0])
    check(_lib.lib.tg_check_range(ptr(e), n, int(state.num_edges), stream_ptr()))
    hits = t.empty(n, dtype=t.bool, device=e.device)
    feats = None
    store = state.c_store()
    if state.features is not None:
        feats = padded_rows((n,), int(state.features.shape[1]), e.device, zero=False)
    check(_lib.lib.tg_cache_lookup(ptr(e), n, state.c_cache(), ptr(hits), store, ptr(feats),
                                   int(feats.stride(0)) if feats is not None else 0, stream_ptr()))
    h = int(hits.sum().item()) if n else 0
    state.sim_fast_cost += float(h)
    state.sim_slow_cost += float((n - h) * slow_cost_per_row)
    if host:
        return (None if feats is None else feats.cpu().numpy()), hits.cpu().numpy()
    return feats, hits


def maybe_replace(state):
    """Epoch-boundary replacement decision; counters reset either way
    (cache.py:107-118)."""
    state.epoch_stats[-1].close()  # read the epoch's hits/misses before K6 resets them
    out = (_lib.c_int64 * 4)()
    store = state.c_store()
    hot = state.hot
    check(_lib.lib.tg_cache_replace(state.c_cache(), int(state.k), int(state.epsilon), store, ptr(hot),
                                    int(hot.stride(0)) if hot is not None else 0, out, stream_ptr()))
    replaced = bool(out[0])
    state.replacements.append(replaced)
    state.epoch_stats.append(EpochStats(state))
    return replaced


def topk_mask(counts, k):
    """Device top-k of touched counts (count desc, eid asc) as a bool mask."""
    t = _lib.torch()
    c = to_device(counts, t.int32).reshape(-1)
    m = t.empty(c.shape[0], dtype=t.uint8, device=c.device)
    sel = _lib.c_int64(0)
    check(_lib.lib.tg_topk_mask(ptr(c), int(c.shape[0]), int(k), ptr(m), _lib.ctypes.byref(sel), stream_ptr()))
    return m.bool()


def oracle_cache(trace_counts, k):
    """Per-epoch hit rate of the clairvoyant top-k cache (cache.py:121-136)."""
    t = _lib.torch()
    tc = trace_counts if isinstance(trace_counts, t.Tensor) else t.as_tensor(np.asarray(trace_counts))
    rates = []
    for epoch in tc:
        e = epoch.to(device="cuda", dtype=t.int64)
        total = int(e.sum().item())
        if total == 0:
            rates.append(None)
            continue
        m = topk_mask(e, k)
        rates.append(float(int(e[m].sum().item()) / total))
    return rates


def run_trace(state, trace):
    """Feed a per-epoch trace (lists of eids) through the cache; returns
    per-epoch hit rates (cache.py:139-147)."""
    rates = []
    for epoch_eids in trace:
        lookup(state, epoch_eids)
        rates.append(state.epoch_stats[-1].hit_rate())
        maybe_replace(state)
    return rates


def cache_report(state, oracle_rates=None):
    """JSON-ready metrics for the run so far (cache.py:150-176)."""
    epochs = []
    for i, st in enumerate(state.epoch_stats):
        if st.requests == 0 and i == len(state.epoch_stats) - 1:
            break
        epochs.append({
            "epoch": i,
            "requests": st.requests,
            "hits": st.hits,
            "hit_rate": st.hit_rate(),
            "zero_denominator": st.requests == 0,
            "oracle_hit_rate": (oracle_rates[i] if oracle_rates is not None and i < len(oracle_rates) else None),
            "replaced": state.replacements[i] if i < len(state.replacements) else None,
        })
    report = {
        "budget_k": state.k,
        "epsilon": state.epsilon,
        "final_resident_count": state.resident_count,
        "replacement_events": int(sum(state.replacements)),
        "epochs": epochs,
        "simulated_fast_cost": state.sim_fast_cost,
        "simulated_slow_cost": state.sim_slow_cost,
    }
    json.dumps(report)
    return report
