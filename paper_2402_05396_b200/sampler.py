"""Adaptive neighbor sampler: policy sampling without replacement (K8).

Drop-in for sampler.py:43-50 (``PolicyOutput``) and sampler.py:138-176
(``sample_without_replacement``).  The scoring half (encoders, mixer,
decoders, masked softmax -> q, log q) is K7: fused in ``scoring.py`` for the
pipeline, and stage by stage here and in ``encoders.py`` with the
reference's signatures -- ``mixer_transform(z, mask, store)``
(sampler.py:69-72) and ``decode_policy(z_raw, z_mixed, z_target, mask, scfg,
ecfg, store, d_v, d_e)`` (sampler.py:91-135) -- on CUDA tensors in the
store's dtype.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ConfigError, check, ptr, stream_ptr, to_device
from .seeds import device_pcg

DECODER_KINDS = ("linear", "gat", "gatv2", "trans")


@dataclass(frozen=True)
class SamplerConfig:
    decoder: str = "linear"
    n: int = 10
    m: int = 25
    negative_slope: float = 0.2

    def __post_init__(self):
        if self.decoder not in DECODER_KINDS:
            raise ConfigError(f"unknown decoder {self.decoder!r}; expected one of {DECODER_KINDS}")
        if not 1 <= self.n <= self.m:
            raise ConfigError(f"need 1 <= n <= m, got n={self.n} m={self.m}")


@dataclass
class PolicyOutput:
    q: object                  # (B, m), zero on masked slots, sums to 1 over valid
    log_q: object              # (B, m), sentinel on masked slots
    mask: object               # (B, m)
    selected: object = None        # (B, n) slot indices, -1 where unused
    selected_mask: object = None   # (B, n)
    selected_log_q: object = None  # (B, n)


def _dev(x, dtype=None):
    t = _lib.torch()
    if isinstance(x, t.Tensor):
        return x.to(device="cuda").contiguous() if dtype is None else x.to(device="cuda", dtype=dtype).contiguous()
    data = getattr(x, "data", x)  # reference autodiff Tensor exposes .data
    arr = np.ascontiguousarray(np.asarray(data))
    return to_device(arr, dtype if dtype is not None else t.from_numpy(arr).dtype)


def sample_wor_device(q, log_q, n, rng, B_global=None, rows=None, selected=None, sel_mask=None, sel_log_q=None,
                      stream=None):
    """Launch K8 on device tensors; returns (selected, sel_mask, sel_log_q).

    rng: numpy PCG64 Generator positioned where the reference's would be.
    B_global/rows: the batch width of the RNG stream and this shard's rows.
    """
    t = _lib.torch()
    B, m = int(q.shape[0]), int(q.shape[1])
    if q.dtype == t.float64:
        dtype = 1
    elif q.dtype == t.float32:
        dtype = 0
    else:
        raise ValueError("q must be f32 or f64")
    if log_q is not None and log_q.dtype != q.dtype:
        log_q = log_q.to(q.dtype)
    if selected is None:
        selected = t.empty((B, n), dtype=t.int64, device=q.device)
    if sel_mask is None:
        sel_mask = t.empty((B, n), dtype=t.bool, device=q.device)
    if sel_log_q is None and log_q is not None:
        sel_log_q = t.empty((B, n), dtype=q.dtype, device=q.device)
    pcg = device_pcg(rng, B if B_global is None else B_global)
    check(_lib.lib.tg_sample_wor(ptr(q), ptr(log_q), dtype, B, m, int(n), pcg,
                                 rows if rows is not None else _lib.rowmap(), ptr(selected), ptr(sel_mask),
                                 ptr(sel_log_q), stream_ptr(stream)))
    return selected, sel_mask, sel_log_q


def sample_without_replacement(policy, n, rng):
    """Draw up to n distinct valid slots per row by sequential renormalised
    draws from q; records log q of each pick under the original q
    (sampler.py:138-176).  Mutates and returns ``policy``; ``rng`` is
    advanced by exactly the draws the reference would consume."""
    t = _lib.torch()
    host = not isinstance(policy.q, t.Tensor)
    q = _dev(policy.q)
    if q.dtype not in (t.float32, t.float64):
        q = q.to(t.float64)
    lq = _dev(policy.log_q, q.dtype) if policy.log_q is not None else None
    B = int(q.shape[0])
    sel, smask, slq = sample_wor_device(q, lq, n, rng)
    # the reference stops drawing after the first round with no live row
    rounds = int(smask.sum(dim=1).max().item()) if B else 0
    rng.bit_generator.advance(rounds * B)
    if host:
        policy.selected = sel.cpu().numpy()
        policy.selected_mask = smask.cpu().numpy()
        policy.selected_log_q = None if slq is None else slq.cpu().numpy()
    else:
        policy.selected, policy.selected_mask, policy.selected_log_q = sel, smask, slq
    return policy


def _stage_cfg(d_enc, m):
    """An EncoderConfig whose encoded width is d_enc (the mixer stage only
    reads d_enc and m; F and the feature kinds just have to be consistent)."""
    from .encoders import EncoderConfig
    for k, (dv, de) in ((2, (0, 0)), (3, (1, 0)), (4, (1, 1))):
        if d_enc > m and (d_enc - m) % k == 0:
            F = (d_enc - m) // k
            return EncoderConfig.balanced(F, m), dv, de
    raise ValueError(f"width {d_enc} is not an encoded width for scope {m}")


def _as_rows(x, lead, d, dtype):
    """(tensor, row stride) of a [lead, d] CUDA view in `dtype`."""
    t = _lib.torch()
    if not isinstance(x, t.Tensor):
        x = t.as_tensor(np.ascontiguousarray(np.asarray(getattr(x, "data", x))))
    x = x.to(device="cuda", dtype=dtype).reshape(lead, d)
    if x.stride(1) != 1:
        x = x.contiguous()
    return x, int(x.stride(0))


def mixer_transform(z, mask, store, stream=None):
    """One mixer layer over the neighborhood (mixer.py:31-51) with masked
    rows forced to zero (sampler.py:69-72).  z [B, m, d_enc] -> same shape."""
    t = _lib.torch()
    from .encoders import StageModel, padded_out
    B, m, d = (int(x) for x in z.shape)
    ecfg, dv, de = _stage_cfg(d, m)
    sm = StageModel(ecfg, store, dv, de, d_enc=d)
    sm.require("ln1_g", "ln1_b", "Wc1", "bc1", "Wc2", "bc2", "ln2_g", "ln2_b", "Wt1", "bt1", "Wt2", "bt2")
    out = padded_out(B * m, d, sm.dtype)
    if B == 0:
        return out.reshape(B, m, d)
    zz, ldz = _as_rows(z, B * m, d, sm.dtype)
    mk = _dev(mask, t.bool).view(t.uint8)
    ws, nb = sm.workspace(B)
    check(_lib.lib.tg_mixer_transform(sm.c, ptr(zz), ldz, ptr(mk), B, ptr(out), int(out.stride(0)), ptr(ws), nb,
                                      stream_ptr(stream)))
    return out.reshape(B, m, d)


def decode_policy(z_raw, z_mixed, z_target, mask, scfg, ecfg, store, d_v, d_e, stream=None):
    """Per-slot sampling distribution (sampler.py:91-135): logits from the
    decoder of ``scfg``, masked softmax and log-softmax (autodiff.py:429-464).
    Returns PolicyOutput(q, log_q, mask) as CUDA tensors."""
    t = _lib.torch()
    from .encoders import StageModel
    B, m, d = (int(x) for x in z_raw.shape)
    sm = StageModel(ecfg, store, d_v, d_e, decoder=scfg.decoder, negative_slope=scfg.negative_slope)
    if d != sm.d_enc:
        raise ValueError(f"z_raw width {d} != encoded width {sm.d_enc}")
    sm.require({"linear": "w_linear", "gat": "W_gat", "gatv2": "W_gatv2", "trans": "W_trans_target"}[scfg.decoder],
               *({"gat": ["a_gat"], "gatv2": ["a_gatv2"], "trans": ["W_trans_nbr"]}.get(scfg.decoder, [])))
    mk = _dev(mask, t.bool)
    q = t.empty((B, m), dtype=sm.dtype, device="cuda")
    lq = t.empty((B, m), dtype=sm.dtype, device="cuda")
    if B == 0:
        return PolicyOutput(q=q, log_q=lq, mask=mk)
    zr, ldr = _as_rows(z_raw, B * m, d, sm.dtype)
    zm, ldm = (None, 0) if z_mixed is None else _as_rows(z_mixed, B * m, d, sm.dtype)
    zt, ldt = (None, 0) if z_target is None else _as_rows(z_target, B, sm.d_tv, sm.dtype)
    ws, nb = sm.workspace(B)
    check(_lib.lib.tg_decode_policy(sm.c, ptr(zr), ldr, ptr(zm), ldm, ptr(zt), ldt, ptr(mk.view(t.uint8)), B, ptr(q),
                                    ptr(lq), ptr(ws), nb, stream_ptr(stream)))
    return PolicyOutput(q=q, log_q=lq, mask=mk)
