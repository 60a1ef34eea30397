"""K7: the adaptive sampler's scoring forward pass on the device.

One call replaces the chain the reference Trainer runs per adaptive layer
(training.py:269-276): ``encode_neighborhood_batch`` (encoders.py:152),
``mixer_transform`` (sampler.py:69), ``encode_target_batch``
(encoders.py:186), ``decode_policy`` (sampler.py:91) with its masked
softmax / log-softmax (autodiff.py:429-464).  Intermediates (z_raw, the
mixer output) stay in a device workspace; the result is the policy's
(q, log q) in the model's precision.

The backward half: ``SamplerGrad`` runs
``tg_score_backward`` -- the scoring network's vjps from d loss / d logits
(K10's output) to every sampler parameter, the ``ad.backward`` of
update_sampler (sampler.py:253-256) -- and ``update_sampler`` applies the
device Adam (optim.AdamState, params.py:80-99) to the model in place.
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


class SamplerGrad:
    """Gradient buffers of a ScoringModel's parameters, accumulated over the
    layers of one update like the reference's ``.grad`` (training.py:411-436:
    the surrogate loss sums every adaptive layer's term)."""

    def __init__(self, model):
        t = _lib.torch()
        self.model = model
        self.grads = {name: t.zeros_like(x) for name, x in model.named_params().items()}
        self._ws = None

    def zero_grad(self):
        for g in self.grads.values():
            g.zero_()

    def grad(self, name):
        """d loss / d parameter in the reference's shape."""
        f = {v: k for k, v in self.model._FIELDS.items()}[name]
        return self.grads[name].view(self.model.shapes[f])

    def backward(self, ids, dts, mask, dlogits, node_rows=None, edge_rows=None, tgt_rows=None, stream=None):
        """Accumulate the gradients of one candidate block (the inputs of the
        ``score_policy`` call that produced the logits) from dlogits [B, m]."""
        t = _lib.torch()
        model = self.model
        B, m = int(ids.shape[0]), int(ids.shape[1])
        if m != model.m:
            raise ValueError(f"batch has scope {m}, config expects {model.m}")
        if tuple(dlogits.shape) != (B, m):
            raise ValueError(f"dlogits must be ({B}, {m}), got {tuple(dlogits.shape)}")
        if B == 0:
            return self
        dl = dlogits.to(device=ids.device, dtype=model.dtype).contiguous()
        nr, nld = _rows(node_rows, B, m, model.d_v)
        er, eld = _rows(edge_rows, B, m, model.d_e)
        tr, tld = _rows(tgt_rows, B, 1, model.d_v)
        n = _lib.ctypes.c_size_t(0)
        check(_lib.lib.tg_score_backward_workspace(model.c, B, _lib.ctypes.byref(n)))
        if self._ws is None or self._ws.numel() < n.value:
            self._ws = t.empty(max(int(n.value), 256), dtype=t.uint8, device=ids.device)
        g = _lib.tg_score_grads()
        inv = {v: k for k, v in model._FIELDS.items()}
        for name, buf in self.grads.items():
            setattr(g, inv[name], ptr(buf))
        mk = mask.view(t.uint8) if mask.dtype == t.bool else mask
        check(_lib.lib.tg_score_backward(model.c, ptr(ids), ptr(dts), ptr(mk.contiguous()), ptr(nr), nld, ptr(er),
                                         eld, ptr(tr), tld, B, ptr(dl), g, ptr(self._ws), int(n.value),
                                         stream_ptr(stream)))
        return self


def update_sampler(sgrad, adam, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """update_sampler (sampler.py:253-256) after the backward: one Adam step
    over the whole sampler store (K10 tg_adam_step, bit-identical to
    ParamStore.adam_step), then the gradients are cleared like adam_step
    clears .grad.  ``adam`` is an optim.AdamState over
    ``sgrad.model.named_params()`` (the tensors K7 reads)."""
    adam.step(sgrad.grads, lr, beta1=beta1, beta2=beta2, eps=eps)
    sgrad.zero_grad()
