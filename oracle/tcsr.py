"""T-CSR construction restated (TEST INFRASTRUCTURE).  Follows graph.py:94-152.

The reference sorts events stably by ts (graph.py:112), reassigns eids
(:131), duplicates each event into both endpoint lists and lexsorts by
(node, ts, eid) (:133-137).  This restatement uses the equivalent
formulation the device kernel relies on -- a stable sort of the interleaved
entries (2*eid + side) by node -- so the golden vectors from the real
reference check that equivalence too.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class DataError(ValueError):
    pass


@dataclass
class OracleGraph:
    num_nodes: int
    src: np.ndarray
    dst: np.ndarray
    ts: np.ndarray
    tcsr_offsets: np.ndarray
    tcsr_neighbors: np.ndarray
    tcsr_ts: np.ndarray
    tcsr_eids: np.ndarray
    node_features: np.ndarray = None
    edge_features: np.ndarray = None

    @property
    def num_events(self):
        return self.src.shape[0]

    @property
    def d_v(self):
        return 0 if self.node_features is None else self.node_features.shape[1]

    @property
    def d_e(self):
        return 0 if self.edge_features is None else self.edge_features.shape[1]


def build_graph(src, dst, ts, num_nodes=None, node_features=None, edge_features=None):
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    ts = np.asarray(ts, dtype=np.float64)
    if not (src.shape == dst.shape == ts.shape):
        raise DataError("src/dst/ts length mismatch")
    if ts.size and not np.isfinite(ts).all():
        raise DataError("non-finite timestamp")
    if ts.size and (ts < 0).any():
        raise DataError("negative timestamp")
    if src.size and ((src < 0).any() or (dst < 0).any()):
        raise DataError("negative node id")
    perm = np.argsort(ts, kind="stable")                      # graph.py:112
    src, dst, ts = src[perm], dst[perm], ts[perm]
    if edge_features is not None:
        edge_features = np.asarray(edge_features, dtype=np.float32)
        if edge_features.shape[0] != src.shape[0]:
            raise DataError("edge feature row count does not match event count")
        edge_features = edge_features[perm]
    top = int(max(src.max(), dst.max())) + 1 if src.size else 0
    if num_nodes is None:
        num_nodes = top
    elif num_nodes < top:
        raise DataError(f"num_nodes={num_nodes} smaller than max node id {top - 1}")
    if node_features is not None:
        node_features = np.asarray(node_features, dtype=np.float32)
        if node_features.shape[0] != num_nodes:
            raise DataError("node feature row count does not match num_nodes")
    E = src.shape[0]
    # entry 2e+side: side 0 lives in src[e]'s list (peer dst[e]), side 1 in dst[e]'s
    owner = np.empty(2 * E, dtype=np.int64)
    owner[0::2], owner[1::2] = src, dst
    peer = np.empty(2 * E, dtype=np.int64)
    peer[0::2], peer[1::2] = dst, src
    by_node = np.argsort(owner, kind="stable")                # (node, eid) order
    eid_of = by_node >> 1
    counts = np.bincount(owner, minlength=num_nodes) if E else np.zeros(num_nodes, dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return OracleGraph(num_nodes=int(num_nodes), src=src, dst=dst, ts=ts, tcsr_offsets=offsets,
                       tcsr_neighbors=peer[by_node], tcsr_ts=ts[eid_of], tcsr_eids=eid_of.astype(np.int64),
                       node_features=node_features, edge_features=edge_features)


# ---------------------------------------------------------------------------
# Size-independent T-CSR check for graphs too large to rebuild on the host
# ---------------------------------------------------------------------------

def _check_kernel():
    import os
    os.environ.setdefault("NUMBA_THREADING_LAYER", "workqueue")
    from numba import njit, prange

    @njit(parallel=True, cache=False)
    def kern(src, dst, ts, offsets, nbr, tts, eid, bad):
        V = offsets.shape[0] - 1
        for v in prange(V):
            nb = 0
            prev = -1
            for k in range(offsets[v], offsets[v + 1]):
                e = np.int64(eid[k])
                ok = 0 <= e < src.shape[0]
                if ok:
                    s, d = src[e], dst[e]
                    ok = (s == v or d == v) and nbr[k] == (d if s == v else s) and tts[k] == ts[e]
                    # (node, ts, eid) order = eid order when ts is non-decreasing in eid;
                    # an eid repeats only as a self-loop's two entries
                    if e < prev:
                        ok = False
                    elif e == prev and (s != d or (k - 2 >= offsets[v] and eid[k - 2] == e)):
                        ok = False
                if not ok:
                    nb += 1
                prev = e
            bad[v] = nb
    return kern


_KERN = None


def check_tcsr(src, dst, ts, offsets, nbr, tts, eid):
    """Number of T-CSR entries that differ from graph.py:94-152's output for
    the events (src, dst, ts) -- without re-sorting 2E entries.  Valid for
    event arrays in eid order with ts non-decreasing (build_graph's output
    order).  Per node v the reference holds every event incident to v once
    (a self-loop twice), ordered by (ts, eid); so the device T-CSR is
    identical iff (1) offsets == [0, cumsum(bincount(src) + bincount(dst))],
    (2) every entry of v's segment names an event incident to v, its peer and
    its ts, (3) eids ascend within the segment, repeating only for a
    self-loop's two entries.  (1)-(3) admit exactly one arrangement."""
    global _KERN
    V = offsets.shape[0] - 1
    if not (np.diff(ts) >= 0).all():
        raise ValueError("check_tcsr needs events in non-decreasing ts order")
    deg = np.bincount(src, minlength=V) + np.bincount(dst, minlength=V)
    want = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(deg, out=want[1:])
    off_bad = int((want != offsets).sum())
    if off_bad:
        return off_bad, int(offsets[-1])
    if _KERN is None:
        _KERN = _check_kernel()
    bad = np.zeros(V, dtype=np.int64)
    _KERN(src, dst, ts, offsets, nbr, tts, eid, bad)
    return int(bad.sum()), int(offsets[-1])
