"""Synthetic graphs of the five BASELINE.json shapes, generated on the device.

SURVEY §8(d): src ~ Zipf(1.2) over a seeded node permutation (the idea of
synth.py:63-68, vectorised), dst uniform, ts sorted-uniform over [0, 1e6)
(or tie-heavy / integer variants), f32 features from a counter hash in
[-1, 1).  Every value is a pure function of the seed, so oracle/shapes.py
rebuilds identical host copies for the parity checks.  The GDELT shape
(191M events, 142 GB of 186-d rows) is written straight into HBM by
tg_synth_* -- no host staging.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr
from .graph import build_graph, padded_rows
from .pipeline import PathConfig  # noqa: F401  (re-export)
from .specs import SHAPES, ShapeSpec  # noqa: F401  (re-export)

ZIPF_S = 1.2
SPAN = 1.0e6


def zipf_tables(V, seed, s=ZIPF_S):
    """(cdf f64[V], node_at_rank int64[V]) shared by host and device."""
    w = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w / w.sum())
    node_at_rank = np.random.default_rng([int(seed), 0x5EED]).permutation(V).astype(np.int64)
    return cdf, node_at_rank


def feature_seeds(seed):
    return 2 * int(seed) + 1, 2 * int(seed) + 2  # (edge, node)


def synth_events_device(V, E, seed, ts_mode=0, span=SPAN, device=None):
    t = _lib.torch()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    cdf, nar = zipf_tables(V, seed)
    cdf_d = t.as_tensor(cdf).to(dev)
    nar_d = t.as_tensor(nar).to(dev)
    src = t.empty(E, dtype=t.int64, device=dev)
    dst = t.empty(E, dtype=t.int64, device=dev)
    ts = t.empty(E, dtype=t.float64, device=dev)
    check(_lib.lib.tg_synth_events(0, E, E, V, int(seed), ptr(cdf_d), ptr(nar_d), int(ts_mode), float(span),
                                   ptr(src), ptr(dst), ptr(ts), stream_ptr()))
    return src, dst, ts


def synth_features_device(rows, d, seed, device=None, out=None, chunk=1 << 24, row0=0):
    """Rows [row0, row0 + rows) of the hash-defined table (out row i = row row0 + i)."""
    t = _lib.torch()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if out is None:
        out = padded_rows((rows,), d, dev)
    for r0 in range(0, rows, chunk):
        n = min(chunk, rows - r0)
        check(_lib.lib.tg_synth_features(row0 + r0, n, int(d), int(seed), ptr(out[r0:]), int(out.stride(0)),
                                         stream_ptr()))
    return out


def sharded_features(rows, d, seed, group=None):
    """Collective: this rank's shard of the hash-defined table, peers mapped
    over CUDA IPC (placement.ShardedTable)."""
    from .placement import ShardedTable

    def fill(own, lo, hi):
        synth_features_device(hi - lo, d, seed, out=own, row0=lo)

    return ShardedTable.from_process_group(rows, d, fill, group=group)


def make_graph(spec, seed=0, ts_mode=0, device=None, features=True, edge_placement="replicated"):
    """Device TemporalGraph of a ShapeSpec (events -> K1 T-CSR -> features).
    edge_placement "sharded": the edge table is split by eid range across
    the ranks of the default process group (collective; placement.py)."""
    if edge_placement not in ("replicated", "sharded"):
        raise ValueError(f"unknown edge placement {edge_placement!r}")
    t = _lib.torch()
    src, dst, ts = synth_events_device(spec.V, spec.E, seed, ts_mode, device=device)
    eseed, nseed = feature_seeds(seed)
    ef = None
    if features and spec.d_e and ts_mode != 0:
        ef = synth_features_device(spec.E, spec.d_e, eseed, device=src.device)
    g = build_graph(src, dst, ts, num_nodes=spec.V, edge_features=ef)
    del src, dst, ts
    if features and spec.d_e and edge_placement == "sharded":
        if ef is not None:
            raise ValueError("sharded placement needs the sorted generator (ts_mode 0)")
        t.cuda.synchronize()
        t.cuda.empty_cache()
        g.edge_features = sharded_features(spec.E, spec.d_e, eseed)
    elif features and spec.d_e and ts_mode == 0:
        # sorted generator: eid == generation index, write rows in eid order
        t.cuda.synchronize()
        t.cuda.empty_cache()  # release the build's sort temporaries before the big table
        g.edge_features = synth_features_device(spec.E, spec.d_e, eseed, device=g.device)
    if features and spec.d_v:
        g.node_features = synth_features_device(spec.V, spec.d_v, nseed, device=g.device)
    return g
