"""Host twin of the synthetic shape generator (TEST INFRASTRUCTURE).

Regenerates, with numpy uint64/f64 arithmetic, exactly what
paper_2402_05396_b200/csrc/synth.cu writes on the device, so small shapes can
be built on both sides and compared bit-for-bit, and the CPU baseline can be
timed on the same data.
"""

from __future__ import annotations

import os

import numpy as np

from .rng import GOLDEN, STREAM, mix_np
from .tcsr import build_graph

ZIPF_S = 1.2
SPAN = 1.0e6


def zipf_tables(V, seed, s=ZIPF_S):
    w = 1.0 / np.arange(1, V + 1, dtype=np.float64) ** s
    cdf = np.cumsum(w / w.sum())
    node_at_rank = np.random.default_rng([int(seed), 0x5EED]).permutation(V).astype(np.int64)
    return cdf, node_at_rank


def _hstream(seed, stream, c):
    with np.errstate(over="ignore"):
        key = mix_np(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) * np.uint64(STREAM)))
        return mix_np(key + (np.asarray(c, dtype=np.uint64) + np.uint64(1)) * np.uint64(GOLDEN))


def _unit(z):
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def synth_events(V, E, seed, ts_mode=0, span=SPAN, threads=None, chunk=1 << 22):
    """(src, dst, ts) of the device generator (synth.cu).  Large E is done in
    event chunks on a thread pool (numpy releases the GIL in its loops), so
    the GDELT-shaped 191M events take seconds rather than a minute."""
    cdf, nar = zipf_tables(V, seed)
    src = np.empty(E, dtype=np.int64)
    dst = np.empty(E, dtype=np.int64)
    ts = np.empty(E, dtype=np.float64)

    def part(e0):
        e1 = min(E, e0 + chunk)
        e = np.arange(e0, e1, dtype=np.uint64)
        rank = np.searchsorted(cdf, _unit(_hstream(seed, 1, e)), side="left")
        src[e0:e1] = nar[np.minimum(rank, V - 1)]
        dst[e0:e1] = (_hstream(seed, 2, e) % np.uint64(V)).astype(np.int64)
        if ts_mode == 0:
            ts[e0:e1] = (e.astype(np.float64) + _unit(_hstream(seed, 3, e))) * (span / float(E))
        elif ts_mode == 1:
            ts[e0:e1] = np.floor(_unit(_hstream(seed, 4, e)) * float(E // 8 if E // 8 > 0 else 1))
        else:
            ts[e0:e1] = e.astype(np.float64) + 1.0

    starts = range(0, E, chunk)
    if E > chunk:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads or os.cpu_count() or 1) as pool:
            list(pool.map(part, starts))
    else:
        for e0 in starts:
            part(e0)
    return src, dst, ts


def synth_features(r0, n, d, seed, chunk=1 << 18):
    """Rows [r0, r0 + n) of the hash-defined feature table (synth.cu)."""
    return synth_feature_rows(np.arange(r0, r0 + n, dtype=np.uint64), d, seed, chunk)


def synth_feature_rows(rows, d, seed, chunk=1 << 18):
    """Rows `rows` (any order) of the hash-defined feature table: the parity
    checks regenerate only the rows a mini-batch touched."""
    rows = np.asarray(rows).astype(np.uint64)
    n = rows.shape[0]
    if n > chunk:  # bound the uint64 temporaries (n x d x 8 B each)
        out = np.empty((n, d), dtype=np.float32)
        for c0 in range(0, n, chunk):
            out[c0:c0 + chunk] = synth_feature_rows(rows[c0:c0 + chunk], d, seed, chunk)
        return out
    with np.errstate(over="ignore"):
        key = mix_np(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF) ^ ((rows + np.uint64(1)) * np.uint64(STREAM)))
        j = np.arange(1, d + 1, dtype=np.uint64)
        z = mix_np(key[:, None] + j[None, :] * np.uint64(GOLDEN))
    hi = (z >> np.uint64(40)).astype(np.int64) - 8388608
    return hi.astype(np.float32) * np.float32(1.0 / 8388608.0)


def feature_seeds(seed):
    return 2 * int(seed) + 1, 2 * int(seed) + 2


def make_graph(spec, seed=0, ts_mode=0, features=True):
    src, dst, ts = synth_events(spec.V, spec.E, seed, ts_mode)
    eseed, nseed = feature_seeds(seed)
    ef = synth_features(0, spec.E, spec.d_e, eseed) if (features and spec.d_e) else None
    nf = synth_features(0, spec.V, spec.d_v, nseed) if (features and spec.d_v) else None
    return build_graph(src, dst, ts, num_nodes=spec.V, node_features=nf, edge_features=ef)


class HashRows:
    """Read-only stand-in for a hash-defined feature table too large for host
    RAM (GDELT: 142 GB): indexing with an eid array regenerates exactly those
    rows, so the oracle pipeline can check a full-size mini-batch."""

    def __init__(self, n, d, seed, threads=None):
        self.shape = (int(n), int(d))
        self.dtype = np.dtype(np.float32)
        self.seed = seed
        self.threads = threads or os.cpu_count() or 1

    def __getitem__(self, idx):
        idx = np.asarray(idx)
        if idx.dtype == bool:
            idx = np.flatnonzero(idx)
        flat = idx.ravel().astype(np.int64)
        if flat.size and (flat.min() < 0 or flat.max() >= self.shape[0]):
            raise IndexError("row out of range")
        out = np.empty((flat.size, self.shape[1]), dtype=np.float32)
        chunk = 1 << 15
        if flat.size > chunk:
            from concurrent.futures import ThreadPoolExecutor

            def part(c0):
                out[c0:c0 + chunk] = synth_feature_rows(flat[c0:c0 + chunk], self.shape[1], self.seed)

            with ThreadPoolExecutor(self.threads) as pool:
                list(pool.map(part, range(0, flat.size, chunk)))
        else:
            out[:] = synth_feature_rows(flat, self.shape[1], self.seed)
        return out.reshape(idx.shape + (self.shape[1],))


def synth_events_at(V, E, seed, eids, ts_mode=0, span=SPAN):
    """(src, dst, ts) of the events `eids` of synth_events(V, E, seed)."""
    e = np.asarray(eids).astype(np.uint64)
    cdf, nar = zipf_tables(V, seed)
    rank = np.searchsorted(cdf, _unit(_hstream(seed, 1, e)), side="left")
    src = nar[np.minimum(rank, V - 1)]
    dst = (_hstream(seed, 2, e) % np.uint64(V)).astype(np.int64)
    if ts_mode == 0:
        ts = (e.astype(np.float64) + _unit(_hstream(seed, 3, e))) * (span / float(E))
    elif ts_mode == 1:
        ts = np.floor(_unit(_hstream(seed, 4, e)) * float(E // 8 if E // 8 > 0 else 1))
    else:
        ts = e.astype(np.float64) + 1.0
    return src, dst, ts
