"""Event-file ingest restated (TEST INFRASTRUCTURE).

Follows graph.py:159-205 of the reference: ``ingest_events`` reads
``src,dst,ts[,f...]`` lines (Python text mode: universal newlines),
strips each, skips blank and '#' lines, parses int/int/float/float...,
rejects non-finite timestamps and inconsistent feature widths with
``path:lineno: ...`` messages.  Returns the raw arrays (before
build_graph) so the device parser can be compared field by field.
"""

from __future__ import annotations

import numpy as np


class DataError(ValueError):
    pass


def ingest_arrays(path, d_e=None):
    srcs, dsts, tss, feats = [], [], [], []
    width = d_e
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split(",")
            if len(parts) < 3:
                raise DataError(f"{path}:{lineno}: expected at least src,dst,ts")
            try:
                s, d = int(parts[0]), int(parts[1])
                t = float(parts[2])
                f = [float(x) for x in parts[3:]]
            except ValueError as exc:
                raise DataError(f"{path}:{lineno}: {exc}") from None
            if not np.isfinite(t):
                raise DataError(f"{path}:{lineno}: non-finite timestamp {parts[2]!r}")
            if width is None:
                width = len(f)
            elif len(f) != width:
                raise DataError(f"{path}:{lineno}: edge feature width {len(f)} != expected {width}")
            srcs.append(s)
            dsts.append(d)
            tss.append(t)
            feats.append(f)
    width = width or 0
    ef = np.array(feats, dtype=np.float32).reshape(len(srcs), width) if width else None
    return (np.array(srcs, dtype=np.int64), np.array(dsts, dtype=np.int64), np.array(tss, dtype=np.float64), ef)


def line_error(path, lineno, line, width):
    """The DataError text the reference raises for one failing line."""
    line = line.strip()
    parts = line.split(",")
    if len(parts) < 3:
        return f"{path}:{lineno}: expected at least src,dst,ts"
    try:
        int(parts[0]), int(parts[1])
        t = float(parts[2])
        f = [float(x) for x in parts[3:]]
    except ValueError as exc:
        return f"{path}:{lineno}: {exc}"
    if not np.isfinite(t):
        return f"{path}:{lineno}: non-finite timestamp {parts[2]!r}"
    if width is not None and len(f) != width:
        return f"{path}:{lineno}: edge feature width {len(f)} != expected {width}"
    return None
