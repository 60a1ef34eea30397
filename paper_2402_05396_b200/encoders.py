"""Reference-signature drop-ins for the sampler's encoders (encoders.py).

``encode_neighborhood_batch(ids, dts, mask, node_rows, edge_rows, cfg, store)``
(encoders.py:152-183) and ``encode_target_batch(ids, node_rows, cfg, store)``
(encoders.py:186-200) with the reference's arguments: an ``EncoderConfig``
and a ParamStore-like mapping (``store[name]`` -> array / torch tensor /
object with ``.data``; ``store.dtype`` picks float64 (default) or float32).
They run K7's encoder stage (tg_encode_neighborhood / tg_encode_target,
hand-written kernels + the projections) and return CUDA tensors in the
store's dtype: z [B, m, d_enc] (masked rows exactly zero) and z_t [B, d_tv].
Feature rows are read as float32 (the device tables' type; the reference's
rows are f32 upcast, so the narrowing is exact for them).

The device encoders share one width for features, time and frequency
(``EncoderConfig.balanced``, the reference Trainer's rule,
training.py:153-157); other configurations raise ConfigError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import ConfigError, check, ptr, stream_ptr
from .params import DECODERS, freq_table, omega_table


@dataclass(frozen=True)
class EncoderConfig:
    d_time: int
    d_freq: int
    d_feat: int
    m: int
    alpha: float = None
    beta: float = None

    def __post_init__(self):
        if min(self.d_time, self.d_freq, self.d_feat) < 1 or self.m < 1:
            raise ValueError("encoder dimensions and scope m must be >= 1")
        if self.alpha is None:
            object.__setattr__(self, "alpha", float(np.sqrt(self.d_time)))
        if self.beta is None:
            object.__setattr__(self, "beta", float(np.sqrt(self.d_time)))
        if self.alpha <= 0 or self.beta <= 0:
            raise ValueError("time-encoding constants must be positive")

    @classmethod
    def balanced(cls, dim, m, alpha=None, beta=None):
        return cls(d_time=dim, d_freq=dim, d_feat=dim, m=m, alpha=alpha, beta=beta)


def encoded_width(cfg, d_v, d_e):
    """d_enc (encoders.py:116-119)."""
    return (cfg.d_feat if d_v else 0) + (cfg.d_feat if d_e else 0) + cfg.d_time + cfg.d_freq + cfg.m


def target_width(cfg, d_v):
    """d_tv (encoders.py:122-123)."""
    return (cfg.d_feat if d_v else 0) + cfg.d_time + cfg.d_freq


# ---------------------------------------------------------------------------
# store -> tg_score_model
# ---------------------------------------------------------------------------

_FIELDS = {"W_node": "encoder/W_node", "W_edge": "encoder/W_edge", "ln1_g": "sampler/mixer/ln1_gamma",
           "ln1_b": "sampler/mixer/ln1_beta", "Wc1": "sampler/mixer/Wc1", "bc1": "sampler/mixer/bc1",
           "Wc2": "sampler/mixer/Wc2", "bc2": "sampler/mixer/bc2", "ln2_g": "sampler/mixer/ln2_gamma",
           "ln2_b": "sampler/mixer/ln2_beta", "Wt1": "sampler/mixer/Wt1", "bt1": "sampler/mixer/bt1",
           "Wt2": "sampler/mixer/Wt2", "bt2": "sampler/mixer/bt2", "w_linear": "sampler/w_linear",
           "W_gat": "sampler/W_gat", "a_gat": "sampler/a_gat", "W_gatv2": "sampler/W_gatv2",
           "a_gatv2": "sampler/a_gatv2", "W_trans_target": "sampler/W_trans_target",
           "W_trans_nbr": "sampler/W_trans_nbr"}


def store_dtype(store):
    t = _lib.torch()
    dt = getattr(store, "dtype", np.float64)
    if dt in (t.float32, np.float32) or str(dt) in ("float32", "torch.float32"):
        return t.float32
    return t.float64


def _lookup(store, name):
    try:
        return store[name]
    except (KeyError, IndexError):
        return None


def _param(store, name, dtype, dev):
    """One store entry as a contiguous CUDA tensor of `dtype` (no copy when
    it already is one)."""
    t = _lib.torch()
    x = _lookup(store, name)
    if x is None:
        return None
    if not isinstance(x, t.Tensor):
        x = t.as_tensor(np.ascontiguousarray(np.asarray(getattr(x, "data", x))))
    return x.to(device=dev, dtype=dtype).contiguous()


class StageModel:
    """tg_score_model over a store's parameters for one (cfg, widths, decoder)."""

    def __init__(self, ecfg, store, d_v, d_e, decoder="linear", negative_slope=0.2, d_enc=None):
        t = _lib.torch()
        _lib.require_cuda("the sampler's encoders / mixer / decoders")
        if not (ecfg.d_time == ecfg.d_freq == ecfg.d_feat):
            raise ConfigError("the device encoders need d_time == d_freq == d_feat (EncoderConfig.balanced)")
        self.dtype = store_dtype(store)
        dev = t.device("cuda", t.cuda.current_device())
        F, m = int(ecfg.d_feat), int(ecfg.m)
        self.F, self.m, self.d_v, self.d_e = F, m, int(d_v), int(d_e)
        self.d_enc = encoded_width(ecfg, d_v, d_e) if d_enc is None else int(d_enc)
        self.d_tv = target_width(ecfg, d_v)
        self._keep = {}
        c = _lib.tg_score_model()
        c.dtype = 1 if self.dtype == t.float64 else 0
        c.decoder = DECODERS[decoder]
        c.m, c.F, c.d_v, c.d_e = m, F, self.d_v, self.d_e
        c.d_enc, c.d_tv, c.slope, c.gemm_path = self.d_enc, self.d_tv, float(negative_slope), 1
        for field, name in _FIELDS.items():
            x = _param(store, name, self.dtype, dev)
            if x is not None:
                self._keep[field] = x
                setattr(c, field, ptr(x))
        self._keep["omega"] = t.as_tensor(omega_table(F, float(ecfg.alpha), float(ecfg.beta))).to(dev)
        self._keep["fe_table"] = t.as_tensor(freq_table(m, F)).to(dev)
        c.omega, c.fe_table = ptr(self._keep["omega"]), ptr(self._keep["fe_table"])
        self.c = c
        self.dev = dev

    def require(self, *fields):
        missing = [_FIELDS[f] for f in fields if f not in self._keep]
        if missing:
            raise ConfigError(f"sampler parameters missing: {missing}")

    def workspace(self, B):
        t = _lib.torch()
        n = _lib.ctypes.c_size_t(0)
        check(_lib.lib.tg_score_stage_workspace(self.c, int(B), _lib.ctypes.byref(n)))
        return t.empty(max(int(n.value), 256), dtype=t.uint8, device=self.dev), int(n.value)


def rows_f32(x, lead, d):
    """Feature rows as a 16-byte-pitched f32 [n, d] CUDA matrix (None if d == 0)."""
    t = _lib.torch()
    if x is None or d == 0:
        return None, 0
    if not isinstance(x, t.Tensor):
        x = t.as_tensor(np.ascontiguousarray(np.asarray(getattr(x, "data", x))))
    x = x.to(device="cuda", dtype=t.float32).reshape(lead, d)
    if x.stride(1) != 1 or x.stride(0) % 4 or x.data_ptr() % 16:
        from .graph import padded_rows
        y = padded_rows((lead,), d, x.device)
        y.copy_(x)
        x = y
    return x, int(x.stride(0))


def _dev(x, dtype):
    t = _lib.torch()
    if not isinstance(x, t.Tensor):
        x = t.as_tensor(np.ascontiguousarray(np.asarray(getattr(x, "data", x))))
    return x.to(device="cuda", dtype=dtype).contiguous()


def padded_out(lead, d, dtype):
    """[lead, d] view of a [lead, round4(d)] buffer (16-B rows, like K7's)."""
    t = _lib.torch()
    ld = (d + 3) & ~3
    return t.zeros((lead, ld), dtype=dtype, device="cuda")[:, :d]


def encode_neighborhood_batch(ids, dts, mask, node_rows, edge_rows, cfg, store, stream=None):
    """z [B, m, d_enc] for a padded candidate batch (encoders.py:152-183):
    [GeLU(x_v W_node) | GeLU(x_e W_edge) | cos(dt w) | FE(freq) | identity],
    masked rows exactly zero."""
    t = _lib.torch()
    ids_d = _dev(ids, t.int64)
    B, m = int(ids_d.shape[0]), int(ids_d.shape[1])
    if m != cfg.m:
        raise ValueError(f"batch has scope {m}, config expects {cfg.m}")
    d_v = 0 if node_rows is None else int(node_rows.shape[-1])
    d_e = 0 if edge_rows is None else int(edge_rows.shape[-1])
    sm = StageModel(cfg, store, d_v, d_e)
    sm.require(*(["W_node"] if d_v else []), *(["W_edge"] if d_e else []))
    out = padded_out(B * m, sm.d_enc, sm.dtype)
    if B == 0:
        return out.reshape(B, m, sm.d_enc)
    nr, nld = rows_f32(node_rows, B * m, d_v)
    er, eld = rows_f32(edge_rows, B * m, d_e)
    ws, nb = sm.workspace(B)
    mk = _dev(mask, t.bool).view(t.uint8)
    check(_lib.lib.tg_encode_neighborhood(sm.c, ptr(ids_d), ptr(_dev(dts, t.float64)), ptr(mk), ptr(nr), nld, ptr(er),
                                          eld, B, ptr(out), int(out.stride(0)), ptr(ws), nb, stream_ptr(stream)))
    return out.reshape(B, m, sm.d_enc)


def encode_target_batch(ids, node_rows, cfg, store, stream=None):
    """z_t [B, d_tv] = [GeLU(x_v W_node) | TE(0) | FE(1)] (encoders.py:186-200)."""
    t = _lib.torch()
    B = int(np.asarray(ids).shape[0]) if not isinstance(ids, t.Tensor) else int(ids.shape[0])
    d_v = 0 if node_rows is None else int(node_rows.shape[-1])
    sm = StageModel(cfg, store, d_v, 0)
    if d_v:
        sm.require("W_node")
    out = padded_out(B, sm.d_tv, sm.dtype)
    if B == 0:
        return out
    tr, tld = rows_f32(node_rows, B, d_v)
    ws, nb = sm.workspace(B)
    check(_lib.lib.tg_encode_target(sm.c, ptr(tr), tld, B, ptr(out), int(out.stride(0)), ptr(ws), nb,
                                    stream_ptr(stream)))
    return out
