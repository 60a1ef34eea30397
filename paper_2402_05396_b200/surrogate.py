"""Surrogate-loss head of the sampler update on the device (K10).

Drop-in for the surrogate losses of sampler.py:183-250 as the reference's
Trainer composes them (training.py:409-436), SURVEY §8(f) rank 3:

  tgat_sample_coefficients(dL_dh, tau, V, sel_mask, contrib_mask)      (:191-213)
  graphmixer_sample_coefficients(dL_dh, w_prime, mu, sel_mask, contrib_mask)  (:230-239)
  graphmixer_message_coefficients(dL_dh, msgs, Wc1, Wt1, Wt2, ...)     (training.py:423-431)
  sample_loss_tgat / sample_loss_graphmixer                            (:216-227, 242-250)

The reference returns an autodiff Tensor whose ``backward`` reaches the
scoring logits; here the loss comes back together with that gradient,
d loss / d logits [B, m] (index + log_softmax_masked vjp, autodiff.py:257-271,
447-464) -- the input of the scoring network's backward.  Coefficients are
frozen (no gradient flows into dL_dh, tau, V, mu), as in the reference.
All arrays are CUDA tensors (numpy accepted and copied up); float dtype
follows dL_dh (float32 or float64).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from ._lib import check, ptr, stream_ptr, to_device


@dataclass
class SurrogateGrad:
    loss: object       # f64 CUDA scalar tensor: sum(c * selected_log_q)
    dlogits: object    # (B, m) d loss / d logits, the scoring network's upstream gradient
    c: object          # (B, n) the frozen per-pick coefficients


def _dtype(x):
    t = _lib.torch()
    if isinstance(x, t.Tensor):
        dt = x.dtype
    else:
        import numpy as np
        dt = t.float32 if np.asarray(x).dtype == np.float32 else t.float64
    if dt not in (t.float32, t.float64):
        raise ValueError("float32 or float64 expected")
    return dt, (0 if dt == t.float32 else 1)


def _masks(sel_mask, contrib_mask, B, n):
    t = _lib.torch()
    sm = t.ones((B, n), dtype=t.uint8, device="cuda") if sel_mask is None else to_device(sel_mask, t.bool).to(t.uint8)
    cm = t.ones((B,), dtype=t.uint8, device="cuda") if contrib_mask is None else to_device(contrib_mask, t.bool).to(t.uint8)
    if tuple(sm.shape) != (B, n) or tuple(cm.shape) != (B,):
        raise ValueError("sel_mask must be (B, n) and contrib_mask (B,)")
    return sm.contiguous(), cm.contiguous()


def tgat_sample_coefficients(dL_dh, tau, V, sel_mask=None, contrib_mask=None):
    """Per-pick coefficients of the attention aggregator (sampler.py:191-213).
    FloatingPointError if an active row's normalizer is not positive."""
    t = _lib.torch()
    _lib.require_cuda("tgat_sample_coefficients")
    dt, code = _dtype(dL_dh)
    g, ta, v = to_device(dL_dh, dt), to_device(tau, dt), to_device(V, dt)
    B, n = ta.shape
    d = g.shape[1]
    if tuple(v.shape) != (B, n, d) or g.shape[0] != B:
        raise ValueError("shapes: dL_dh (B, d), tau (B, n), V (B, n, d)")
    sm, cm = _masks(sel_mask, contrib_mask, B, n)
    c = t.empty((B, n), dtype=dt, device="cuda")
    check(_lib.lib.tg_tgat_sample_coeffs(code, B, n, d, ptr(g), d, ptr(ta), ptr(v), ptr(sm), ptr(cm), ptr(c),
                                         stream_ptr()))
    return c


def graphmixer_sample_coefficients(dL_dh, w_prime, mu, sel_mask=None, contrib_mask=None):
    """c_j = (1/n) sum_k dL/dh_k w'_jk mu_jk (sampler.py:230-239); w_prime
    (n, d) or (B, n, d)."""
    t = _lib.torch()
    _lib.require_cuda("graphmixer_sample_coefficients")
    dt, code = _dtype(dL_dh)
    g, m = to_device(dL_dh, dt), to_device(mu, dt)
    B, n, d = m.shape
    wp = to_device(w_prime, dt)
    if wp.dim() == 3 and wp.stride(0) == 0:
        wp = wp[0]
    wp = wp.contiguous()
    if tuple(wp.shape) == (n, d):
        bstride = 0
    elif tuple(wp.shape) == (B, n, d):
        bstride = n * d
    else:
        raise ValueError("w_prime must be (n, d) or (B, n, d)")
    sm, cm = _masks(sel_mask, contrib_mask, B, n)
    c = t.empty((B, n), dtype=dt, device="cuda")
    check(_lib.lib.tg_mixer_sample_coeffs(code, B, n, d, ptr(g), d, ptr(wp), bstride, ptr(m), ptr(sm), ptr(cm),
                                          ptr(c), stream_ptr()))
    return c


def graphmixer_message_coefficients(dL_dh, msgs, Wc1, Wt1, Wt2, sel_mask=None, contrib_mask=None):
    """The Trainer's composition (training.py:423-431): mu = msgs @ Wc1 and
    w'_j = 1 + rowsum(Wt1 @ Wt2)_j, without materialising the (B, n, d) mu."""
    t = _lib.torch()
    _lib.require_cuda("graphmixer_message_coefficients")
    dt, code = _dtype(dL_dh)
    g, ms = to_device(dL_dh, dt), to_device(msgs, dt)
    w1, t1, t2 = to_device(Wc1, dt), to_device(Wt1, dt), to_device(Wt2, dt)
    B, n, dm = ms.shape
    d = g.shape[1]
    ht = t1.shape[1]
    if tuple(w1.shape) != (dm, d) or tuple(t1.shape) != (n, ht) or tuple(t2.shape) != (ht, n):
        raise ValueError("shapes: msgs (B, n, d_msg), Wc1 (d_msg, d), Wt1 (n, ht), Wt2 (ht, n)")
    sm, cm = _masks(sel_mask, contrib_mask, B, n)
    c = t.empty((B, n), dtype=dt, device="cuda")
    check(_lib.lib.tg_graphmixer_sample_coeffs(code, B, n, dm, d, ht, ptr(g), d, ptr(ms), dm, ptr(w1), ptr(t1),
                                               ptr(t2), ptr(sm), ptr(cm), ptr(c), stream_ptr()))
    return c


def surrogate_grad(c, policy):
    """loss = sum(c * selected_log_q) and d loss / d logits for a policy that
    went through sample_without_replacement (its q, log_q, mask, selected,
    selected_mask)."""
    t = _lib.torch()
    _lib.require_cuda("surrogate_grad")
    dt, code = _dtype(c)
    q, lq = to_device(policy.q, dt), to_device(policy.log_q, dt)
    mask = to_device(policy.mask, t.bool).to(t.uint8).contiguous()
    sel = to_device(policy.selected, t.int64)
    sm = to_device(policy.selected_mask, t.bool).to(t.uint8).contiguous()
    cc = to_device(c, dt)
    B, m = q.shape
    n = sel.shape[1]
    dlogits = t.empty((B, m), dtype=dt, device="cuda")
    rows = t.empty((max(B, 1),), dtype=t.float64, device="cuda")
    loss = t.empty((), dtype=t.float64, device="cuda")
    check(_lib.lib.tg_logq_surrogate_grad(code, B, m, n, ptr(q), ptr(lq), ptr(mask), ptr(sel), ptr(sm), ptr(cc),
                                          ptr(dlogits), ptr(rows), ptr(loss), stream_ptr()))
    return SurrogateGrad(loss, dlogits, cc)


def sample_loss_tgat(dL_dh, tau, V, policy, sel_mask=None, contrib_mask=None):
    """sample_loss_tgat (sampler.py:216-227) + its logits gradient; like the
    reference, sel_mask=None means every pick counts."""
    return surrogate_grad(tgat_sample_coefficients(dL_dh, tau, V, sel_mask, contrib_mask), policy)


def sample_loss_graphmixer(dL_dh, w_prime, mu, policy, sel_mask=None, contrib_mask=None):
    """sample_loss_graphmixer (sampler.py:242-250) + its logits gradient."""
    return surrogate_grad(graphmixer_sample_coefficients(dL_dh, w_prime, mu, sel_mask, contrib_mask), policy)
