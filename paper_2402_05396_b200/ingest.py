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

_FEW, _NONFINITE, _WIDTH, _RANGE = 0xFFEF, 0xFFF0, 0xFFF1, 0xFFF4


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


def _patch_long_decimals(raw, path, lines, first, row, width, src, dst, ts, feats):
    """Lines holding a value of more than 19 significant digits whose
    correctly rounded double the device parser cannot settle from its
    truncated significand: parse them here exactly as graph.py:170-179 does
    (int() / float(), in Python) and write the results into the device
    arrays.  Only lines before the device's first failing line matter.
    Returns (line, message) of the first such line Python rejects, else None."""
    t = _lib.torch()
    text = raw.tobytes().decode("utf-8", errors="replace")
    all_lines = text.replace("\r\n", "\n").replace("\r", "\n").split("\n")
    for l in lines:
        if first is not None and l > first:
            break
        line = all_lines[l] if l < len(all_lines) else ""
        msg = _error_text(path, l + 1, line, width)
        if msg is not None:
            return l, msg
        parts = line.strip().split(",")
        s, d = int(parts[0]), int(parts[1])
        if not (-(1 << 63) <= s < (1 << 63) and -(1 << 63) <= d < (1 << 63)):
            return l, f"{path}:{l + 1}: node id outside int64"
        r = int(row[l].item())
        src[r], dst[r] = s, d
        ts[r] = float(parts[2])
        if width:
            feats[r] = t.as_tensor(np.array([float(x) for x in parts[3:]], dtype=np.float32)).to(feats.device)
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
    err = (ctypes.c_int64 * 3)()
    cap = 1024
    while True:
        unsup = t.empty(cap, dtype=t.int64, device=dev)
        check(_lib.lib.tg_ingest_parse(ptr(text), n, ptr(ends), nterm, nlines, ptr(isdata), ptr(nf), ptr(row),
                                       width, ptr(src), ptr(dst), ptr(ts), ptr(feats),
                                       int(feats.stride(0)) if feats is not None else 0, ptr(unsup), cap, err, st))
        if int(err[2]) <= cap:
            break
        cap = int(err[2])  # more undecidable lines than slots: parse again with room for all
    first = int(err[0]) if err[0] >= 0 else None
    fail = None
    if int(err[2]):
        fail = _patch_long_decimals(raw, path, sorted(unsup[:int(err[2])].tolist()), first, row, width,
                                    src, dst, ts, feats)
    if fail is not None and (first is None or fail[0] <= first):
        raise DataError(fail[1])
    if first is not None:
        line = _nth_line(raw.tobytes(), first)
        lineno = first + 1
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
