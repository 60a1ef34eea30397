"""K7: the adaptive sampler's scoring forward pass on the device.

One call replaces the chain the reference Trainer runs per adaptive layer
(training.py:269-276): ``encode_neighborhood_batch`` (encoders.py:152),
``mixer_transform`` (sampler.py:69), ``encode_target_batch``
(encoders.py:186), ``decode_policy`` (sampler.py:91) with its masked
softmax / log-softmax (autodiff.py:429-464).  Intermediates (z_raw, the
mixer output) stay in a device workspace; the result is the policy's
(q, log q) in the model's precision.
"""

from __future__ import annotations

from . import _lib
from ._lib import check, ptr, stream_ptr


def _rows(x, B, m, d):
    """f32 [B*m, d] view of a feature block (None when the width is 0)."""
    if x is None or d == 0:
        return None, 0
    t = _lib.torch()
    x = x.reshape(-1, d)
    if x.dtype != t.float32 or x.stride(1) != 1 or x.stride(0) % 4 or x.data_ptr() % 16:
        # the tensor-core GEMM reads rows in 16-byte units: re-pitch
        from .graph import padded_rows
        y = padded_rows((int(x.shape[0]),), d, x.device)
        y.copy_(x)
        x = y
    return x, int(x.stride(0))


def score_policy(model, ids, dts, mask, node_rows=None, edge_rows=None, tgt_rows=None, q=None, log_q=None,
                 stream=None):
    """(q, log_q) [B, m] for candidate blocks already on the device.

    ids int64 [B,m], dts f64 [B,m], mask bool/u8 [B,m]; node_rows [B,m,d_v] /
    edge_rows [B,m,d_e] f32 with masked slots zero (training.py:218, 227);
    tgt_rows [B, d_v] the roots' node rows (encoders.py:186).
    """
    t = _lib.torch()
    B, m = int(ids.shape[0]), int(ids.shape[1])
    if m != model.m:
        raise ValueError(f"batch has scope {m}, config expects {model.m}")
    if q is None:
        q = t.empty((B, m), dtype=model.dtype, device=ids.device)
    if log_q is None:
        log_q = t.empty((B, m), dtype=model.dtype, device=ids.device)
    if B == 0:
        return q, log_q
    nr, nld = _rows(node_rows, B, m, model.d_v)
    er, eld = _rows(edge_rows, B, m, model.d_e)
    tr, tld = _rows(tgt_rows, B, 1, model.d_v)
    ws, nbytes = model.workspace(B)
    mk = mask.view(t.uint8) if mask.dtype == t.bool else mask
    check(_lib.lib.tg_score(model.c, ptr(ids), ptr(dts), ptr(mk), ptr(nr), nld, ptr(er), eld, ptr(tr), tld, B,
                            ptr(q), ptr(log_q), ptr(ws), nbytes, stream_ptr(stream)))
    return q, log_q
