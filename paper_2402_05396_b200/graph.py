"""Device-resident temporal graph: the T-CSR built on the GPU (K1).

Mirrors graph.py:50-152 of the reference (``TemporalGraph``,
``build_graph``) and graph.py:266-271 (``temporal_neighborhood_size``) with
the same argument meaning, validation order and ``DataError`` messages.  The
arrays live in HBM as torch tensors:

  src/dst int64[E], ts f64[E]      events in eid order (= stable ts order)
  tcsr_offsets int64[V+1]          per-node ranges
  nbr int32[2E], adj_ts f64[2E], adj_eid int32[2E]   entries sorted (ts, eid)

``tcsr_neighbors``/``tcsr_eids`` return int64 views for reference-typed
callers; kernels read the int32 arrays (half the random-read bytes).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import DataError, check, ptr, stream_ptr, to_device


@dataclass
class TemporalGraph:
    num_nodes: int
    src: object
    dst: object
    ts: object
    tcsr_offsets: object
    nbr32: object
    tcsr_ts: object
    eid32: object
    node_features: object = field(default=None)
    edge_features: object = field(default=None)
    # coarse time index (tg_tcsr_coarse), built on first use by c_graph()
    coarse_shift: int = field(default=6)
    _coarse: object = field(default=None, repr=False, compare=False)

    @property
    def num_events(self):
        return int(self.src.shape[0])

    @property
    def d_v(self):
        return 0 if self.node_features is None else int(self.node_features.shape[1])

    @property
    def d_e(self):
        return 0 if self.edge_features is None else int(self.edge_features.shape[1])

    @property
    def tcsr_neighbors(self):
        return self.nbr32.to(_lib.torch().int64)

    @property
    def tcsr_eids(self):
        return self.eid32.to(_lib.torch().int64)

    @property
    def device(self):
        return self.src.device

    def degree(self, v):
        o = self.tcsr_offsets[v:v + 2].cpu()
        return int(o[1] - o[0])

    def adjacency(self, v):
        o = self.tcsr_offsets[v:v + 2].cpu()
        lo, hi = int(o[0]), int(o[1])
        t = _lib.torch()
        return self.nbr32[lo:hi].to(t.int64), self.tcsr_ts[lo:hi], self.eid32[lo:hi].to(t.int64)

    def c_graph(self):
        """tg_graph view for the C-ABI (pointers stay valid while self lives),
        with the coarse time index (every 2^coarse_shift-th timestamp per node,
        L2-resident) the finder searches hubs through; coarse_shift 0 turns it
        off.  Built once, on the graph's device, the first time it is asked for."""
        g = _lib.tg_graph(ptr(self.tcsr_offsets), ptr(self.nbr32), ptr(self.tcsr_ts), ptr(self.eid32),
                          int(self.num_nodes), int(self.nbr32.shape[0]), None, None, 0, 0)
        if self.coarse_shift and self.nbr32.shape[0] > 0:
            if self._coarse is None:
                t = _lib.torch()
                n = (int(self.nbr32.shape[0]) >> self.coarse_shift) + int(self.num_nodes)
                coff = t.empty(int(self.num_nodes) + 1, dtype=t.int64, device=self.device)
                cts = t.empty(max(n, 1), dtype=t.float64, device=self.device)
                check(_lib.lib.tg_tcsr_coarse(_lib.ctypes.byref(g), int(self.coarse_shift), ptr(coff), ptr(cts),
                                              stream_ptr()))
                t.cuda.current_stream(self.device).synchronize()  # before finders on any stream read it
                self._coarse = (coff, cts)
            g.coarse_off, g.coarse_ts = ptr(self._coarse[0]), ptr(self._coarse[1])
            g.coarse_shift = int(self.coarse_shift)
        return g

    def edge_store(self):
        return feat_store(self.edge_features)

    def node_store(self):
        return feat_store(self.node_features)


def row_pitch(d):
    """Row stride (floats) of feature tables and mini-batch row buffers:
    d rounded up to 16 bytes so K5 moves rows in 16-byte units and the rows
    are TMA-addressable."""
    return (int(d) + 3) & ~3


def padded_rows(shape, d, device, zero=True):
    """[*shape, d] f32 view of a [*shape, row_pitch(d)] buffer."""
    t = _lib.torch()
    pitch = row_pitch(d)
    buf = (t.zeros if zero else t.empty)((*shape, pitch), dtype=t.float32, device=device)
    return buf[..., :d] if pitch != d else buf


def as_padded_table(x):
    """A [rows, d] f32 CUDA table with row stride row_pitch(d) (copy if needed)."""
    if x is None:
        return None
    d = int(x.shape[1])
    if x.stride(1) == 1 and x.stride(0) == row_pitch(d):
        return x
    out = padded_rows((int(x.shape[0]),), d, x.device)
    out.copy_(x)
    return out


def feat_store(table, hot=None, hot_ld=0):
    """tg_feat_store over a [rows, d] f32 CUDA table (None -> width 0)."""
    if table is None:
        return _lib.tg_feat_store(None, None, None, 0, 0, 0, 0, 0, 0)
    if hasattr(table, "c_store"):  # placement.ShardedTable
        return table.c_store(hot, hot_ld)
    return _lib.tg_feat_store(ptr(table), ptr(hot), None, 0, 0, int(table.shape[1]), int(table.stride(0)),
                              int(hot_ld), int(table.shape[0]))


def build_graph(src, dst, ts, num_nodes=None, node_features=None, edge_features=None, device=None):
    """Assemble a device TemporalGraph from parallel event arrays.

    Same contract as graph.py:94-152: events are re-ordered by (ts, input
    position), eids reassigned to match, feature rows follow their events.
    """
    t = _lib.torch()
    _lib.require_cuda("build_graph")
    src = to_device(src, t.int64, device)
    dst = to_device(dst, t.int64, device)
    ts = to_device(ts, t.float64, device)
    if not (src.shape == dst.shape == ts.shape) or src.dim() != 1:
        raise DataError("src/dst/ts length mismatch")
    E = int(src.shape[0])
    info = (_lib.c_int64 * 2)()
    st = stream_ptr()
    check(_lib.lib.tg_tcsr_check(ptr(src), ptr(dst), ptr(ts), E, info, st))
    max_node, ts_sorted = int(info[0]), int(info[1])

    if edge_features is not None:
        edge_features = to_device(edge_features, t.float32, src.device, rows_ok=True)
        if edge_features.dim() != 2 or edge_features.shape[0] != E:
            raise DataError("edge feature row count does not match event count")

    inferred = max_node + 1 if E else 0
    if num_nodes is None:
        num_nodes = inferred
    elif num_nodes < inferred:
        raise DataError(f"num_nodes={num_nodes} smaller than max node id {inferred - 1}")
    num_nodes = int(num_nodes)
    if node_features is not None:
        node_features = to_device(node_features, t.float32, src.device, rows_ok=True)
        if node_features.dim() != 2 or node_features.shape[0] != num_nodes:
            raise DataError("node feature row count does not match num_nodes")
        node_features = as_padded_table(node_features)

    dev = src.device
    order = t.empty(E, dtype=t.int64, device=dev) if (edge_features is not None and not ts_sorted) else None
    src_s = t.empty(E, dtype=t.int64, device=dev)
    dst_s = t.empty(E, dtype=t.int64, device=dev)
    ts_s = t.empty(E, dtype=t.float64, device=dev)
    offsets = t.empty(num_nodes + 1, dtype=t.int64, device=dev)
    nbr = t.empty(2 * E, dtype=t.int32, device=dev)
    adj_ts = t.empty(2 * E, dtype=t.float64, device=dev)
    adj_eid = t.empty(2 * E, dtype=t.int32, device=dev)
    check(_lib.lib.tg_tcsr_build(ptr(src), ptr(dst), ptr(ts), E, num_nodes, ts_sorted, ptr(order), ptr(src_s),
                                 ptr(dst_s), ptr(ts_s), ptr(offsets), ptr(nbr), ptr(adj_ts), ptr(adj_eid), st))
    if edge_features is not None and order is not None:
        d = int(edge_features.shape[1])
        permuted = padded_rows((E,), d, dev)
        check(_lib.lib.tg_gather_rows_f32(ptr(edge_features), int(edge_features.stride(0)), ptr(order), E, d,
                                          ptr(permuted), int(permuted.stride(0)), st))
        edge_features = permuted
    elif edge_features is not None:
        edge_features = as_padded_table(edge_features)
    return TemporalGraph(num_nodes=num_nodes, src=src_s, dst=dst_s, ts=ts_s, tcsr_offsets=offsets, nbr32=nbr,
                         tcsr_ts=adj_ts, eid32=adj_eid, node_features=node_features, edge_features=edge_features)


def from_device_tcsr(num_nodes, src, dst, ts, offsets, nbr32, adj_ts, eid32, node_features=None,
                     edge_features=None):
    """Wrap already-built device arrays (used by the synthetic shape path)."""
    return TemporalGraph(num_nodes=int(num_nodes), src=src, dst=dst, ts=ts, tcsr_offsets=offsets, nbr32=nbr32,
                         tcsr_ts=adj_ts, eid32=eid32, node_features=node_features, edge_features=edge_features)


def temporal_neighborhood_size(graph, v, t):
    """Number of interactions of ``v`` strictly before ``t`` (graph.py:266-271)."""
    if not 0 <= v < graph.num_nodes:
        raise DataError(f"node id {v} out of range")
    from .finder import pivot
    return pivot(graph, v, t)


def graphs_equal(a, b):
    """Structural equality, features bit-for-bit (graph.py:290-304)."""
    t = _lib.torch()
    if a.num_nodes != b.num_nodes or a.num_events != b.num_events:
        return False
    for name in ("src", "dst", "ts", "tcsr_offsets", "nbr32", "tcsr_ts", "eid32"):
        if not t.equal(getattr(a, name), getattr(b, name)):
            return False
    for name in ("node_features", "edge_features"):
        fa, fb = getattr(a, name), getattr(b, name)
        if (fa is None) != (fb is None):
            return False
        if fa is not None and not t.equal(fa.view(t.int32), fb.view(t.int32)):
            return False
    return True


def as_numpy(x):
    if x is None:
        return None
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
