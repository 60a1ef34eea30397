"""Event files straight into a device T-CSR.

Drop-in for graph.py:159-222 of the reference: ``ingest_events(path, d_e,
num_nodes, node_feature_path)`` and ``load_manifest(path)``.  The file's
bytes are copied to HBM once and parsed by ingest.cu (line scan, warp per
line, CPython int()/float() semantics with correct rounding); the events
then go through K1 (build_graph) without leaving the device.  Errors are
the reference's DataError messages for the first failing line.
"""

from __future__ import annotations

import ctypes
import json
import os
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import DataError, check, ptr, stream_ptr
from .graph import build_graph, padded_rows
from .matio import load_features_device

_FEW, _NONFINITE, _WIDTH, _UNSUP, _RANGE = 0xFFEF, 0xFFF0, 0xFFF1, 0xFFF3, 0xFFF4


def _nth_line(raw, index):
    """Line `index` (0-based) of the file in Python's universal-newline split."""
    text = raw.decode("utf-8", errors="replace")
    lines = text.replace("\r\n", "\n").replace("\r", "\n").split("\n")  # text-mode universal newlines
    return lines[index] if index < len(lines) else ""


def _error_text(path, lineno, line, width):
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
    if len(f) != width:
        return f"{path}:{lineno}: edge feature width {len(f)} != expected {width}"
    return None


def ingest_arrays_device(path, d_e=None, device=None):
    """(src, dst, ts, edge_features | None) CUDA tensors of an event file."""
    t = _lib.torch()
    _lib.require_cuda("ingest_events")
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    path = Path(path)
    raw = np.fromfile(path, dtype=np.uint8)
    n = int(raw.size)
    text = t.from_numpy(raw).pin_memory().to(dev, non_blocking=True) if n else t.empty(1, dtype=t.uint8,
                                                                                         device=dev)
    st = stream_ptr()
    info = (ctypes.c_int64 * 4)()
    check(_lib.lib.tg_ingest_lines(ptr(text), n, None, info, st))
    nterm, nlines = int(info[0]), int(info[1])
    ends = t.empty(max(nterm, 1), dtype=t.int64, device=dev)
    check(_lib.lib.tg_ingest_lines(ptr(text), n, ptr(ends), info, st))
    isdata = t.empty(max(nlines, 1), dtype=t.int32, device=dev)
    nf = t.empty_like(isdata)
    row = t.empty_like(isdata)
    check(_lib.lib.tg_ingest_classify(ptr(text), n, ptr(ends), nterm, nlines, ptr(isdata), ptr(nf), ptr(row), info,
                                      st))
    ndata, first, nf0 = int(info[0]), int(info[1]), int(info[2])
    width = int(d_e) if d_e is not None else (nf0 - 3 if first >= 0 and nf0 >= 3 else 0)
    src = t.empty(ndata, dtype=t.int64, device=dev)
    dst = t.empty(ndata, dtype=t.int64, device=dev)
    ts = t.empty(ndata, dtype=t.float64, device=dev)
    feats = padded_rows((max(ndata, 1),), width, dev, zero=False) if width > 0 else None
    err = (ctypes.c_int64 * 2)()
    check(_lib.lib.tg_ingest_parse(ptr(text), n, ptr(ends), nterm, nlines, ptr(isdata), ptr(nf), ptr(row), width,
                                   ptr(src), ptr(dst), ptr(ts), ptr(feats),
                                   int(feats.stride(0)) if feats is not None else 0, err, st))
    if err[0] >= 0:
        line = _nth_line(raw.tobytes(), int(err[0]))
        lineno = int(err[0]) + 1
        if err[1] == _UNSUP:
            raise ValueError(f"{path}:{lineno}: a value with more than 19 significant digits could not be "
                             "rounded on the device")
        if err[1] == _RANGE:
            raise DataError(f"{path}:{lineno}: node id outside int64")
        msg = _error_text(path, lineno, line, width)
        raise DataError(msg or f"{path}:{lineno}: malformed line")
    if feats is not None and ndata == 0:
        feats = feats[:0]
    return src, dst, ts, feats


def ingest_events(path, d_e=None, num_nodes=None, node_feature_path=None, device=None):
    """graph.py:159-205 on the device: parse, then K1 (build_graph)."""
    src, dst, ts, ef = ingest_arrays_device(path, d_e=d_e, device=device)
    node_features = None
    if node_feature_path is not None:
        node_features = load_features_device(node_feature_path, device=device)
        if node_features.shape[1] == 0:
            node_features = None
    return build_graph(src, dst, ts, num_nodes=num_nodes, node_features=node_features, edge_features=ef,
                       device=device)


def load_manifest(path, device=None):
    """graph.py:208-222: the manifest's event + feature files."""
    path = Path(path)
    with open(path) as fh:
        spec = json.load(fh)
    base = path.parent
    node_path = spec.get("node_features")
    g = ingest_events(base / spec["events"], d_e=spec.get("d_e"), num_nodes=spec.get("num_nodes"),
                      node_feature_path=(base / node_path) if node_path else None, device=device)
    if spec.get("d_v") is not None and g.d_v != spec["d_v"]:
        raise DataError(f"manifest d_v={spec['d_v']} but node features have width {g.d_v}")
    if spec.get("d_e") is not None and g.d_e != spec["d_e"]:
        raise DataError(f"manifest d_e={spec['d_e']} but edge features have width {g.d_e}")
    return g
