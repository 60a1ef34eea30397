"""Sampler parameters: the reference ParamStore's values, resident on the device.

The reference keys every initial value by (store seed, crc32(name))
(params.py:19-21, glorot-uniform :56-61) and creates the sampler's tensors
in init_encoder_params (encoders.py:126-130) / init_sampler_params
(sampler.py:53-66) order.  ``sampler_params`` reproduces those arrays on the
host (parameter initialisation, not the per-batch path); ``from_arrays``
takes any name -> array mapping instead (e.g. a trained ParamStore's
``{n: store[n].data}``).  ``ScoringModel`` uploads them once in the compute
dtype and exposes the C-ABI struct ``tg_score_model``.
"""

from __future__ import annotations

import zlib

import numpy as np

from . import _lib
from ._lib import ConfigError, ptr

DECODERS = {"linear": 0, "gat": 1, "gatv2": 2, "trans": 3}


def _glorot(seed, name, shape):
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), zlib.crc32(name.encode("utf-8"))]))
    fan_in, fan_out = (shape[0], shape[-1]) if len(shape) > 1 else (shape[0], shape[0])
    limit = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-limit, limit, size=shape)


def encoded_width(enc_dim, m, d_v, d_e):
    """encoders.py:116-119."""
    return (enc_dim if d_v else 0) + (enc_dim if d_e else 0) + 2 * enc_dim + m


def target_width(enc_dim, d_v):
    """encoders.py:122-123."""
    return (enc_dim if d_v else 0) + 2 * enc_dim


def sampler_params(store_seed, enc_dim, m, d_v, d_e, decoder):
    """name -> float64 array, equal to a fresh reference sampler store."""
    if decoder not in DECODERS:
        raise ConfigError(f"unknown decoder {decoder!r}; expected one of {tuple(DECODERS)}")
    d = encoded_width(enc_dim, m, d_v, d_e)
    p = {}
    if d_v:
        p["encoder/W_node"] = _glorot(store_seed, "encoder/W_node", (d_v, enc_dim))
    if d_e:
        p["encoder/W_edge"] = _glorot(store_seed, "encoder/W_edge", (d_e, enc_dim))
    pre = "sampler/mixer"
    for ln in ("ln1", "ln2"):
        p[f"{pre}/{ln}_gamma"] = np.ones(d)
        p[f"{pre}/{ln}_beta"] = np.zeros(d)
    p[f"{pre}/Wc1"] = _glorot(store_seed, f"{pre}/Wc1", (d, d))
    p[f"{pre}/bc1"] = np.zeros(d)
    p[f"{pre}/Wc2"] = _glorot(store_seed, f"{pre}/Wc2", (d, d))
    p[f"{pre}/bc2"] = np.zeros(d)
    p[f"{pre}/Wt1"] = _glorot(store_seed, f"{pre}/Wt1", (m, m))
    p[f"{pre}/bt1"] = np.zeros(m)
    p[f"{pre}/Wt2"] = _glorot(store_seed, f"{pre}/Wt2", (m, m))
    p[f"{pre}/bt2"] = np.zeros(m)
    shapes = {"linear": {"sampler/w_linear": (d, 1)},
              "gat": {"sampler/W_gat": (d, d), "sampler/a_gat": (2 * d, 1)},
              "gatv2": {"sampler/W_gatv2": (2 * d, d), "sampler/a_gatv2": (d, 1)},
              "trans": {"sampler/W_trans_target": (target_width(enc_dim, d_v), d),
                        "sampler/W_trans_nbr": (d, d)}}[decoder]
    for name, shape in shapes.items():
        p[name] = _glorot(store_seed, name, shape)
    return p


def encoder_constants(enc_dim, time_span):
    """(alpha, beta) of the Trainer's EncoderConfig (training.py:145-157;
    EncoderConfig.balanced default sqrt(d_time), encoders.py:33-36)."""
    if time_span and time_span > 2.0:
        beta = (enc_dim - 1) / np.log10(time_span) if enc_dim > 1 else 1.0
        return 10.0, max(beta, 1e-3)
    return float(np.sqrt(enc_dim)), float(np.sqrt(enc_dim))


def omega_table(enc_dim, alpha, beta):
    """Time-encoding frequencies alpha^(-(i-1)/beta) (encoders.py:57-59)."""
    i = np.arange(1, enc_dim + 1, dtype=np.float64)
    return alpha ** (-(i - 1.0) / beta)


def freq_table(m, d):
    """freq_encode_array rows for multiplicities 0..m (encoders.py:75-85):
    the multiplicity is an integer in [0, m], so the device indexes this
    table instead of evaluating cos/sin per slot."""
    pairs = (d + 1) // 2
    i = np.arange(1, pairs + 1, dtype=np.float64)
    angle = np.arange(m + 1, dtype=np.float64)[:, None] / np.power(10000.0, 2.0 * i / d)
    out = np.empty((m + 1, 2 * pairs))
    out[:, 0::2] = np.cos(angle)
    out[:, 1::2] = np.sin(angle)
    return np.ascontiguousarray(out[:, :d])


class ScoringModel:
    """Device copy of the sampler parameters in the compute dtype."""

    _FIELDS = {"W_node": "encoder/W_node", "W_edge": "encoder/W_edge", "ln1_g": "sampler/mixer/ln1_gamma",
               "ln1_b": "sampler/mixer/ln1_beta", "Wc1": "sampler/mixer/Wc1", "bc1": "sampler/mixer/bc1",
               "Wc2": "sampler/mixer/Wc2", "bc2": "sampler/mixer/bc2", "ln2_g": "sampler/mixer/ln2_gamma",
               "ln2_b": "sampler/mixer/ln2_beta", "Wt1": "sampler/mixer/Wt1", "bt1": "sampler/mixer/bt1",
               "Wt2": "sampler/mixer/Wt2", "bt2": "sampler/mixer/bt2", "w_linear": "sampler/w_linear",
               "W_gat": "sampler/W_gat", "a_gat": "sampler/a_gat", "W_gatv2": "sampler/W_gatv2",
               "a_gatv2": "sampler/a_gatv2", "W_trans_target": "sampler/W_trans_target",
               "W_trans_nbr": "sampler/W_trans_nbr"}

    def __init__(self, params, decoder, enc_dim, m, d_v, d_e, alpha, beta, precision="float32",
                 negative_slope=0.2, device=None, tensor_cores=None):
        t = _lib.torch()
        _lib.require_cuda("the adaptive sampler")
        if decoder not in DECODERS:
            raise ConfigError(f"unknown decoder {decoder!r}; expected one of {tuple(DECODERS)}")
        if precision not in ("float32", "float64"):
            raise ConfigError(f"unknown precision {precision!r}")
        self.decoder, self.enc_dim, self.m, self.d_v, self.d_e = decoder, int(enc_dim), int(m), int(d_v), int(d_e)
        self.alpha, self.beta, self.precision = float(alpha), float(beta), precision
        self.dtype = t.float64 if precision == "float64" else t.float32
        self.d_enc = encoded_width(self.enc_dim, self.m, self.d_v, self.d_e)
        self.d_tv = target_width(self.enc_dim, self.d_v)
        dev = device if device is not None else t.device("cuda", t.cuda.current_device())
        self._t = {}
        self.shapes = {}
        for field, name in self._FIELDS.items():
            if name in params:
                arr = np.ascontiguousarray(np.asarray(params[name], dtype=np.float64))
                self.shapes[field] = arr.shape
                self._t[field] = t.as_tensor(arr).to(device=dev, dtype=self.dtype).reshape(-1).contiguous()
        self._t["omega"] = t.as_tensor(omega_table(self.enc_dim, self.alpha, self.beta)).to(dev)
        self._t["fe_table"] = t.as_tensor(freq_table(self.m, self.enc_dim)).to(dev)
        need = {"linear": ["w_linear"], "gat": ["W_gat", "a_gat"], "gatv2": ["W_gatv2", "a_gatv2"],
                "trans": ["W_trans_target", "W_trans_nbr"]}[decoder]
        need += ["Wc1", "bc1", "Wc2", "bc2", "Wt1", "bt1", "Wt2", "bt2", "ln1_g", "ln1_b", "ln2_g", "ln2_b"]
        need += (["W_node"] if d_v else []) + (["W_edge"] if d_e else [])
        missing = [self._FIELDS[f] for f in need if f not in self._t]
        if missing:
            raise ConfigError(f"sampler parameters missing: {missing}")
        c = _lib.tg_score_model()
        c.dtype = 1 if self.dtype == t.float64 else 0
        c.decoder = DECODERS[decoder]
        c.m, c.F, c.d_v, c.d_e = self.m, self.enc_dim, self.d_v, self.d_e
        c.d_enc, c.d_tv, c.slope = self.d_enc, self.d_tv, float(negative_slope)
        # f32 GEMMs run on the tcgen05 tensor cores (3xTF32).  The tensor core's
        # fp32 accumulator truncates (measured: ~2.5x the error of an FFMA GEMM
        # at K=328, scripts/diag_tc_acc.py), which the linear / gat / gatv2
        # decoders absorb (q within 6e-6 of f64) but the trans decoder's
        # bilinear logits amplify past 1e-5, so trans keeps FFMA GEMMs.
        if tensor_cores is None:
            tensor_cores = decoder != "trans"
        self.tensor_cores = bool(tensor_cores)
        c.gemm_path = 0 if tensor_cores else 1
        for field, x in self._t.items():
            setattr(c, field, ptr(x))
        self.c = c
        self._ws = None

    def named_params(self):
        """Reference name -> the flat device tensor K7 reads (updated in place
        by an optimizer: the next tg_score call sees the new values)."""
        return {self._FIELDS[f]: x for f, x in self._t.items() if f in self._FIELDS}

    def param(self, name):
        """One parameter as a view in the reference's shape."""
        f = {v: k for k, v in self._FIELDS.items()}[name]
        return self._t[f].view(self.shapes[f])

    def flops(self, B):
        """Algorithmic FLOPs of one tg_score call on B roots (multiply-add = 2):
        feature projections, the mixer the decoder reads, and the decoder."""
        m, d, F = self.m, self.d_enc, self.enc_dim
        f = 2 * B * m * F * (self.d_v + self.d_e)
        if self.decoder in ("linear", "trans"):
            f += 2 * (2 * B * m * d * d) + 2 * (2 * B * d * m * m)
        if self.decoder == "linear":
            f += 2 * B * m * d
        elif self.decoder == "gat":
            f += 2 * B * m * d + 2 * B * d + 4 * d * d
        elif self.decoder == "gatv2":
            f += 2 * B * m * d * d + 2 * B * d * d + 2 * B * m * d
        else:  # reassociated bilinear: u_b = W_n (W_t^T z_t), logits = z_mixed . u_b
            f += 2 * B * self.d_tv * d + 2 * B * d * d + 2 * B * m * d
        return int(f)

    def workspace(self, B):
        t = _lib.torch()
        n = _lib.ctypes.c_size_t(0)
        _lib.check(_lib.lib.tg_score_workspace(self.c, int(B), _lib.ctypes.byref(n)))
        if self._ws is None or self._ws.numel() < n.value:
            self._ws = t.empty(max(int(n.value), 256), dtype=t.uint8, device=self._t["omega"].device)
        return self._ws, int(n.value)
