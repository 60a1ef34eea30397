"""Host twin of the synthetic shape generator (TEST INFRASTRUCTURE).

Regenerates, with numpy uint64/f64 arithmetic, exactly what
paper_2402_05396_b200/csrc/synth.cu writes on the device, so small shapes can
be built on both sides and compared bit-for-bit, and the CPU baseline can be
timed on the same data.
"""

from __future__ import annotations

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


def synth_events(V, E, seed, ts_mode=0, span=SPAN):
    e = np.arange(E, dtype=np.uint64)
    cdf, nar = zipf_tables(V, seed)
    rank = np.searchsorted(cdf, _unit(_hstream(seed, 1, e)), side="left")
    rank = np.minimum(rank, V - 1)
    src = nar[rank]
    dst = (_hstream(seed, 2, e) % np.uint64(V)).astype(np.int64)
    if ts_mode == 0:
        ts = (e.astype(np.float64) + _unit(_hstream(seed, 3, e))) * (span / float(E))
    elif ts_mode == 1:
        ts = np.floor(_unit(_hstream(seed, 4, e)) * float(E // 8 if E // 8 > 0 else 1))
    else:
        ts = e.astype(np.float64) + 1.0
    return src.astype(np.int64), dst, ts


def synth_features(r0, n, d, seed, chunk=1 << 18):
    if n > chunk:  # bound the uint64 temporaries (n x d x 8 B each)
        out = np.empty((n, d), dtype=np.float32)
        for c0 in range(0, n, chunk):
            c = min(chunk, n - c0)
            out[c0:c0 + c] = synth_features(r0 + c0, c, d, seed, chunk)
        return out
    rows = np.arange(r0, r0 + n, dtype=np.uint64)
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
