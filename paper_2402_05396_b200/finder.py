"""Temporal neighbor finder on the device T-CSR (K2).

Drop-in for finder.py of the reference: ``pivot`` (:152), ``batch_find_arrays``
(:162), ``batch_find`` (:192), ``find_recent`` (:209), ``find_uniform`` (:214)
with the same arguments, validation and results.  ``workers`` is accepted
and ignored (the GPU replaces the numba thread pool; results never depended
on it, finder.py:7-9).

Numpy inputs give numpy outputs (exactly the reference's types); torch CUDA
inputs give device tensors without a host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import TG_RECENT, TG_UNIFORM, check, ptr, stream_ptr, to_device


@dataclass(frozen=True)
class NeighborQuery:
    v: int
    t: float
    m: int


@dataclass(frozen=True)
class Neighborhood:
    """Up to m adjacency entries with ts < query.t, most recent first."""

    query: NeighborQuery
    nodes: np.ndarray
    ts: np.ndarray
    eids: np.ndarray

    def __len__(self):
        return self.nodes.shape[0]


_POLICIES = {"recent": TG_RECENT, "uniform": TG_UNIFORM}


def policy_code(policy):
    if policy not in _POLICIES:
        raise ValueError(f"unknown policy {policy!r}")
    return _POLICIES[policy]


def find_args(qv, qt, m, policy, seed, rows=None, seed_ptr=None, **outs):
    """tg_find_args from device tensors; `outs` names the output tensors.
    seed_ptr: optional device u64 (a 0-d view) read by the kernel instead of
    `seed` -- CUDA-graph replays refresh it per batch (pipeline.StepGraph)."""
    a = _lib.tg_find_args()
    a.qv, a.qt, a.B, a.m = ptr(qv), ptr(qt), int(qv.shape[0]), int(m)
    a.policy = policy if isinstance(policy, int) else policy_code(policy)
    a.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    a.rows = rows if rows is not None else _lib.rowmap()
    a.seed_ptr = ptr(seed_ptr)
    for name in ("idx", "cnt", "ids", "eids", "dts", "tss", "mask", "next_v", "next_t", "feat_out", "valid_count",
                 "window"):
        x = outs.get(name)
        setattr(a, name, ptr(x))
    if outs.get("feat_out") is not None:
        a.feat_ld = int(outs["feat_out"].stride(-2))
    return a


def _prepare(qv, qt):
    t = _lib.torch()
    _lib.require_cuda("neighbor finding")
    host = not isinstance(qv, t.Tensor)
    qv_d = to_device(qv, t.int64)
    qt_d = to_device(qt, t.float64)
    return host, qv_d, qt_d


def batch_find_arrays(graph, qv, qt, m, policy="recent", seed=0, workers=None, row_base=0):
    """Vector form of batch_find: (idx, cnt) into the adjacency arrays with
    idx[i, :cnt[i]] the selected entries ts-descending, -1 fill
    (finder.py:162-179).  ``row_base`` offsets the RNG row key (sharding)."""
    t = _lib.torch()
    qv_shape = np.shape(qv) if not isinstance(qv, t.Tensor) else tuple(qv.shape)
    qt_shape = np.shape(qt) if not isinstance(qt, t.Tensor) else tuple(qt.shape)
    if qv_shape != qt_shape:
        raise ValueError("query node/time arrays differ in length")
    if m < 1:
        raise ValueError("budget m must be >= 1")
    code = policy_code(policy)
    host, qv_d, qt_d = _prepare(qv, qt)
    qv_d, qt_d = qv_d.reshape(-1), qt_d.reshape(-1)
    B = int(qv_d.shape[0])
    idx = t.empty((B, m), dtype=t.int64, device=qv_d.device)
    cnt = t.empty(B, dtype=t.int64, device=qv_d.device)
    if B:
        g = graph.c_graph()
        a = find_args(qv_d, qt_d, m, code, seed, rows=_lib.rowmap(None, row_base, 0), idx=idx, cnt=cnt)
        check(_lib.lib.tg_find(g, a, None, None, stream_ptr()))
    if host:
        return idx.cpu().numpy(), cnt.cpu().numpy()
    return idx, cnt


def pivot(graph, v, t):
    """Count of adjacency entries of v with ts strictly < t (finder.py:152-155)."""
    tt = _lib.torch()
    _lib.require_cuda("pivot")
    qv = tt.tensor([int(v)], dtype=tt.int64, device=graph.device)
    qt = tt.tensor([float(t)], dtype=tt.float64, device=graph.device)
    win = tt.empty(1, dtype=tt.int64, device=graph.device)
    a = find_args(qv, qt, 1, TG_RECENT, 0, window=win)
    check(_lib.lib.tg_find(graph.c_graph(), a, None, None, stream_ptr()))
    return int(win.item())


def batch_find(graph, queries, policy="recent", seed=0, workers=None):
    """Neighborhoods for a batch of queries; order matches the input
    (finder.py:192-206).  All queries must share one budget m."""
    if not queries:
        return []
    m = queries[0].m
    if any(q.m != m for q in queries):
        raise ValueError("batch_find requires a single shared budget m")
    tt = _lib.torch()
    qv = tt.tensor([q.v for q in queries], dtype=tt.int64, device=graph.device)
    qt = tt.tensor([q.t for q in queries], dtype=tt.float64, device=graph.device)
    B = len(queries)
    ids = tt.empty((B, m), dtype=tt.int64, device=graph.device)
    eids = tt.empty_like(ids)
    tss = tt.empty((B, m), dtype=tt.float64, device=graph.device)
    cnt = tt.empty(B, dtype=tt.int64, device=graph.device)
    policy_code(policy)
    a = find_args(qv, qt, m, policy, seed, ids=ids, eids=eids, tss=tss, cnt=cnt)
    check(_lib.lib.tg_find(graph.c_graph(), a, None, None, stream_ptr()))
    ids, eids, tss, cnt = ids.cpu().numpy(), eids.cpu().numpy(), tss.cpu().numpy(), cnt.cpu().numpy()
    return [Neighborhood(query=q, nodes=ids[i, :cnt[i]].copy(), ts=tss[i, :cnt[i]].copy(),
                         eids=eids[i, :cnt[i]].copy()) for i, q in enumerate(queries)]


def find_recent(graph, query):
    """The min(m, pivot) most recent valid entries, deterministic."""
    return batch_find(graph, [query], policy="recent")[0]


def find_uniform(graph, query, seed=0):
    """m distinct valid entries, every m-subset equally likely."""
    return batch_find(graph, [query], policy="uniform", seed=seed)[0]


def max_workers():
    """Kept for API parity (finder.py:158); the device has no worker knob."""
    return 1
