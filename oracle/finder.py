"""Temporal neighbor finder restated (TEST INFRASTRUCTURE).

Follows finder.py:69-77 (strict-< pivot), :85-149 (_batch_kernel: recent,
rejection-uniform, complement-uniform with the splitmix64 row stream of
:99-105), :162-179 (batch_find_arrays: -1 / 0 fills).  Compiled with numba
(prange over queries) so that, as the CPU baseline, it runs like the
reference's own numba kernel on all host cores.
"""

from __future__ import annotations

import os

import numpy as np

os.environ.setdefault("NUMBA_THREADING_LAYER", "workqueue")
import numba  # noqa: E402
from numba import njit, prange  # noqa: E402

from .rng import GOLDEN, MIX1, MIX2, STREAM  # noqa: E402

_G = np.uint64(GOLDEN)
_M1 = np.uint64(MIX1)
_M2 = np.uint64(MIX2)
_S = np.uint64(STREAM)


@njit(inline="always")
def _fin(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


@njit(inline="always")
def _lower_bound(ts, lo, hi, t):
    while lo < hi:
        mid = (lo + hi) // 2
        if ts[mid] < t:
            lo = mid + 1
        else:
            hi = mid
    return lo


@njit(inline="always")
def _distinct(key, win, count, buf):
    """First `count` distinct draws of the row stream, in draw order."""
    got = 0
    k = np.uint64(0)
    while got < count:
        k += np.uint64(1)
        r = np.int64(_fin(key + k * _G) % np.uint64(win))
        seen = False
        for j in range(got):
            if buf[j] == r:
                seen = True
                break
        if not seen:
            buf[got] = r
            got += 1


@njit(parallel=True, cache=False)
def _find_kernel(offsets, adj_ts, qv, qt, m, uniform, seed, row_base, idx, cnt, split=np.int64(1 << 62),
                 base1=np.int64(0)):
    for i in prange(qv.shape[0]):
        lo = offsets[qv[i]]
        p = _lower_bound(adj_ts, lo, offsets[qv[i] + 1], qt[i])
        win = p - lo
        if (not uniform) or win <= m:
            c = win if win < m else m
            for j in range(c):
                idx[i, j] = p - 1 - j
            cnt[i] = c
            continue
        grow = row_base + i if i < split else base1 + (i - split)
        key = _fin(np.uint64(seed) ^ (np.uint64(grow) * _S))
        buf = np.empty(m, dtype=np.int64)
        if 2 * m <= win:
            _distinct(key, win, m, buf)
            srt = np.sort(buf)
            for j in range(m):
                idx[i, j] = lo + srt[m - 1 - j]
        else:
            nex = win - m
            _distinct(key, win, nex, buf)
            drop = np.zeros(win, dtype=np.bool_)
            for j in range(nex):
                drop[buf[j]] = True
            k = 0
            for off in range(win - 1, -1, -1):
                if not drop[off]:
                    idx[i, k] = lo + off
                    k += 1
        cnt[i] = m


def batch_find_arrays(graph, qv, qt, m, policy="recent", seed=0, row_base=0, split=None, base1=0):
    """finder.py:162-179; the RNG row key of local query i is row_base + i
    (i < split) or base1 + (i - split) -- the global row under sharding."""
    qv = np.ascontiguousarray(qv, dtype=np.int64)
    qt = np.ascontiguousarray(qt, dtype=np.float64)
    if qv.shape != qt.shape:
        raise ValueError("query node/time arrays differ in length")
    if m < 1:
        raise ValueError("budget m must be >= 1")
    if policy not in ("recent", "uniform"):
        raise ValueError(f"unknown policy {policy!r}")
    idx = np.full((qv.shape[0], m), -1, dtype=np.int64)
    cnt = np.zeros(qv.shape[0], dtype=np.int64)
    _find_kernel(graph.tcsr_offsets, graph.tcsr_ts, qv, qt, int(m), policy == "uniform",
                 np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), np.int64(row_base), idx, cnt,
                 np.int64(1 << 62 if split is None else split), np.int64(base1))
    return idx, cnt


def pivot(graph, v, t):
    lo, hi = graph.tcsr_offsets[v], graph.tcsr_offsets[v + 1]
    return int(np.searchsorted(graph.tcsr_ts[lo:hi], t, side="left"))


def set_threads(n):
    numba.set_num_threads(max(1, min(int(n), numba.config.NUMBA_NUM_THREADS)))


def max_threads():
    return numba.config.NUMBA_NUM_THREADS
