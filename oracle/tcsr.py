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
