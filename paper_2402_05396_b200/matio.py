"""FMAT feature files straight into HBM (first half).

Same on-disk format and errors as matio.py of the reference (:1-59): a
24-byte little-endian header (magic ``b"FMAT"``, u8 version 1, u8 element
code 0 = f32 / 1 = f64, 2 pad bytes, u64 rows, u64 cols) and the row-major
payload.  ``load_features_device`` reads the payload through a pinned
staging buffer in chunks and lands it directly in the 16-byte-pitched
device table the gather kernels use (graph.row_pitch), converting f64 files
to f32 on the device like graph.py:257-259 ``load_features``.  The numpy
functions are provided for API parity.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _lib
from .graph import padded_rows

MAGIC = b"FMAT"
_VERSION = 1
_HEADER = struct.Struct("<4sBBxxQQ")
_DTYPE_CODES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}
_CODE_FOR = {np.dtype("float32"): 0, np.dtype("float64"): 1}


class MatrixFormatError(ValueError):
    """Raised when a matrix file is malformed or truncated (matio.py:23-24)."""


def read_header(path):
    """(dtype, rows, cols) after the reference's checks (matio.py:41-57)."""
    path = Path(path)
    size = path.stat().st_size
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
    if len(head) < _HEADER.size:
        raise MatrixFormatError(f"{path}: file shorter than header")
    magic, version, code, rows, cols = _HEADER.unpack_from(head)
    if magic != MAGIC:
        raise MatrixFormatError(f"{path}: bad magic {magic!r}")
    if version != _VERSION:
        raise MatrixFormatError(f"{path}: unsupported version {version}")
    if code not in _DTYPE_CODES:
        raise MatrixFormatError(f"{path}: unknown element-type code {code}")
    dtype = _DTYPE_CODES[code]
    expected = _HEADER.size + rows * cols * dtype.itemsize
    if size != expected:
        raise MatrixFormatError(
            f"{path}: payload size mismatch (header says {rows}x{cols}, "
            f"{expected - _HEADER.size} bytes, file has {size - _HEADER.size})")
    return dtype, int(rows), int(cols)


def save_matrix(path, array):
    """matio.py:27-36 (a CUDA tensor is copied to the host first)."""
    if hasattr(array, "detach"):
        array = array.detach().cpu().numpy()
    array = np.ascontiguousarray(array)
    if array.ndim != 2:
        raise MatrixFormatError(f"expected a 2-d array, got shape {array.shape}")
    if array.dtype not in _CODE_FOR:
        raise MatrixFormatError(f"unsupported dtype {array.dtype}")
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, _VERSION, _CODE_FOR[array.dtype], array.shape[0], array.shape[1]))
        fh.write(array.astype(array.dtype.newbyteorder("<"), copy=False).tobytes())


def load_matrix(path):
    """matio.py:39-59 on the host (numpy array, native byte order)."""
    dtype, rows, cols = read_header(path)
    data = np.fromfile(path, dtype=dtype, offset=_HEADER.size, count=rows * cols)
    return data.reshape(rows, cols).astype(dtype.newbyteorder("="), copy=True)


def save_features(path, array):
    if hasattr(array, "detach"):
        array = array.detach().cpu().numpy()
    save_matrix(path, np.asarray(array, dtype=np.float32))


def load_features(path):
    return load_matrix(path).astype(np.float32, copy=False)


def load_features_device(path, device=None, chunk_bytes=256 << 20):
    """An FMAT file as a [rows, cols] f32 CUDA table with row pitch
    row_pitch(cols): the payload streams through one pinned chunk buffer
    (H2D copies into the pitched rows); f64 files are narrowed on the device."""
    t = _lib.torch()
    _lib.require_cuda("load_features_device")
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    dtype, rows, cols = read_header(path)
    out = padded_rows((rows,), cols, dev, zero=True)
    if rows == 0 or cols == 0:
        return out
    isz = dtype.itemsize
    per = max(1, chunk_bytes // (cols * isz))
    tdt = t.float32 if isz == 4 else t.float64
    stage = t.empty((min(per, rows), cols), dtype=tdt).pin_memory()
    stage_np = stage.numpy()
    with open(path, "rb") as fh:
        fh.seek(_HEADER.size)
        for r0 in range(0, rows, per):
            n = min(per, rows - r0)
            view = stage_np[:n].reshape(-1).view(np.uint8)
            got = fh.readinto(memoryview(view))
            if got != n * cols * isz:
                raise MatrixFormatError(f"{path}: truncated payload")
            d = stage[:n].to(dev, non_blocking=True)
            out[r0:r0 + n].copy_(d if isz == 4 else d.to(t.float32))
            t.cuda.current_stream().synchronize()  # the staging buffer is reused
    return out
