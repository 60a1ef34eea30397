"""Adaptive-sampler scoring restated in float64 numpy (TEST INFRASTRUCTURE).

The forward half of the TASER policy, as the reference Trainer runs it for
one layer (training.py:269-276):

  encode_neighborhood_batch  encoders.py:152-183 (GeLU projections,
                             cos time encoding :67, frequency encoding
                             :75-85, masked identity block :109-113)
  mixer_transform            sampler.py:69-72 -> mixer.py:31-51
                             (LN autodiff.py:397-418, eps 1e-5, biased var;
                             exact erf GeLU autodiff.py:313-324)
  encode_target_batch        encoders.py:186-200
  decode_policy              sampler.py:91-135 (linear / gat / gatv2 /
                             trans; pad_target_to_neighbor_layout :75-88)
  softmax_masked / log_softmax_masked   autodiff.py:421-464

Parameters follow ParamStore (params.py:19-61): glorot-uniform keyed by
(store seed, crc32(name)), created in the order of init_encoder_params
(encoders.py:126-130) then init_sampler_params (sampler.py:53-66).
Pinned against the real reference by tests/golden/scoring.npz.
"""

from __future__ import annotations

import zlib

import numpy as np
from scipy.special import erf

NEG_INF_LOGIT = -1e30


# ---------------------------------------------------------------- parameters
def _glorot(seed, name, shape):
    rng = np.random.default_rng(np.random.SeedSequence([int(seed), zlib.crc32(name.encode("utf-8"))]))
    fan_in, fan_out = (shape[0], shape[-1]) if len(shape) > 1 else (shape[0], shape[0])
    limit = np.sqrt(6.0 / (fan_in + fan_out))
    return rng.uniform(-limit, limit, size=shape)


def sampler_params(store_seed, enc_dim, m, d_v, d_e, decoder):
    """Every parameter the reference sampler store holds (f64)."""
    d_enc = (enc_dim if d_v else 0) + (enc_dim if d_e else 0) + 2 * enc_dim + m
    d_tv = (enc_dim if d_v else 0) + 2 * enc_dim
    p = {}
    if d_v:
        p["encoder/W_node"] = _glorot(store_seed, "encoder/W_node", (d_v, enc_dim))
    if d_e:
        p["encoder/W_edge"] = _glorot(store_seed, "encoder/W_edge", (d_e, enc_dim))
    pre = "sampler/mixer"
    p[f"{pre}/ln1_gamma"] = np.ones(d_enc)
    p[f"{pre}/ln1_beta"] = np.zeros(d_enc)
    p[f"{pre}/Wc1"] = _glorot(store_seed, f"{pre}/Wc1", (d_enc, d_enc))
    p[f"{pre}/bc1"] = np.zeros(d_enc)
    p[f"{pre}/Wc2"] = _glorot(store_seed, f"{pre}/Wc2", (d_enc, d_enc))
    p[f"{pre}/bc2"] = np.zeros(d_enc)
    p[f"{pre}/ln2_gamma"] = np.ones(d_enc)
    p[f"{pre}/ln2_beta"] = np.zeros(d_enc)
    p[f"{pre}/Wt1"] = _glorot(store_seed, f"{pre}/Wt1", (m, m))
    p[f"{pre}/bt1"] = np.zeros(m)
    p[f"{pre}/Wt2"] = _glorot(store_seed, f"{pre}/Wt2", (m, m))
    p[f"{pre}/bt2"] = np.zeros(m)
    if decoder == "linear":
        p["sampler/w_linear"] = _glorot(store_seed, "sampler/w_linear", (d_enc, 1))
    elif decoder == "gat":
        p["sampler/W_gat"] = _glorot(store_seed, "sampler/W_gat", (d_enc, d_enc))
        p["sampler/a_gat"] = _glorot(store_seed, "sampler/a_gat", (2 * d_enc, 1))
    elif decoder == "gatv2":
        p["sampler/W_gatv2"] = _glorot(store_seed, "sampler/W_gatv2", (2 * d_enc, d_enc))
        p["sampler/a_gatv2"] = _glorot(store_seed, "sampler/a_gatv2", (d_enc, 1))
    elif decoder == "trans":
        p["sampler/W_trans_target"] = _glorot(store_seed, "sampler/W_trans_target", (d_tv, d_enc))
        p["sampler/W_trans_nbr"] = _glorot(store_seed, "sampler/W_trans_nbr", (d_enc, d_enc))
    return p


def encoder_constants(enc_dim, time_span):
    """(alpha, beta) as the Trainer picks them (training.py:145-157,
    encoders.py:33-36)."""
    if time_span and time_span > 2.0:
        beta = (enc_dim - 1) / np.log10(time_span) if enc_dim > 1 else 1.0
        return 10.0, max(beta, 1e-3)
    return float(np.sqrt(enc_dim)), float(np.sqrt(enc_dim))


# ---------------------------------------------------------------- numerics
def gelu(x):
    return x * (0.5 * (1.0 + erf(x * float(1.0 / np.sqrt(2.0)))))


def layer_norm(x, gamma, beta, eps=1e-5):
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return gamma * ((x - mu) * (1.0 / np.sqrt(var + eps))) + beta


def omega(enc_dim, alpha, beta):
    i = np.arange(1, enc_dim + 1, dtype=np.float64)
    return alpha ** (-(i - 1.0) / beta)


def freq_encode(freqs, d):
    pairs = (d + 1) // 2
    i = np.arange(1, pairs + 1, dtype=np.float64)
    angle = np.asarray(freqs, dtype=np.float64)[..., None] / np.power(10000.0, 2.0 * i / d)
    out = np.empty(angle.shape[:-1] + (2 * pairs,))
    out[..., 0::2] = np.cos(angle)
    out[..., 1::2] = np.sin(angle)
    return out[..., :d]


def encode_neighbors(ids, dts, mask, node_rows, edge_rows, p, enc_dim, alpha, beta):
    """z_raw (B, m, d_enc), encoders.py:152-183."""
    B, m = ids.shape
    blocks = []
    for rows, name in ((node_rows, "encoder/W_node"), (edge_rows, "encoder/W_edge")):
        if rows is None or rows.shape[-1] == 0:
            continue
        flat = np.asarray(rows, dtype=np.float64).reshape(B * m, -1) @ p[name]
        blocks.append(gelu(flat).reshape(B, m, enc_dim))
    dv = np.where(mask, dts, 0.0)
    blocks.append(np.cos(dv[..., None] * omega(enc_dim, alpha, beta)))
    ie = (ids[:, :, None] == ids[:, None, :]) & mask[:, :, None] & mask[:, None, :]
    ie = ie.astype(np.float64)
    blocks.append(freq_encode(ie.sum(axis=2), enc_dim))
    blocks.append(ie)
    return np.concatenate(blocks, axis=2) * mask[:, :, None]


def encode_target(node_rows, p, enc_dim, alpha, beta, B):
    """encoders.py:186-200."""
    blocks = []
    if node_rows is not None and node_rows.shape[-1]:
        blocks.append(gelu(np.asarray(node_rows, dtype=np.float64) @ p["encoder/W_node"]))
    blocks.append(np.broadcast_to(np.cos(np.zeros(1)[..., None] * omega(enc_dim, alpha, beta)), (B, enc_dim)))
    blocks.append(np.broadcast_to(freq_encode(np.ones(1), enc_dim), (B, enc_dim)))
    return np.concatenate(blocks, axis=1)


def mixer(z, mask, p, pre="sampler/mixer"):
    """mixer.py:31-51 then the mask (sampler.py:69-72)."""
    B, s, d = z.shape
    x1 = layer_norm(z, p[f"{pre}/ln1_gamma"], p[f"{pre}/ln1_beta"]).reshape(B * s, d)
    h = gelu(x1 @ p[f"{pre}/Wc1"] + p[f"{pre}/bc1"])
    y = z + (h @ p[f"{pre}/Wc2"] + p[f"{pre}/bc2"]).reshape(B, s, d)
    x2 = layer_norm(y, p[f"{pre}/ln2_gamma"], p[f"{pre}/ln2_beta"]).transpose(0, 2, 1).reshape(B * d, s)
    h2 = gelu(x2 @ p[f"{pre}/Wt1"] + p[f"{pre}/bt1"])
    t = (h2 @ p[f"{pre}/Wt2"] + p[f"{pre}/bt2"]).reshape(B, d, s).transpose(0, 2, 1)
    return (y + t) * mask[:, :, None]


def pad_target(zt, enc_dim, m, d_v, d_e):
    B = zt.shape[0]
    off = enc_dim if d_v else 0
    blocks = []
    if off:
        blocks.append(zt[:, :off])
    if d_e:
        blocks.append(np.zeros((B, enc_dim)))
    blocks.append(zt[:, off:off + 2 * enc_dim])
    blocks.append(np.zeros((B, m)))
    return np.concatenate(blocks, axis=1)


def leaky(x, s=0.2):
    return np.where(x > 0.0, x, s * x)


def masked_softmax(logits, mask):
    """(q, log_q), autodiff.py:421-464."""
    neg = np.where(mask, logits, -np.inf)
    mx = neg.max(axis=-1, keepdims=True)
    mx = np.where(np.isfinite(mx), mx, 0.0)
    e = np.exp(np.where(mask, logits - mx, -np.inf))
    z = e.sum(axis=-1, keepdims=True)
    q = np.divide(e, z, out=np.zeros_like(e), where=z > 0)
    lse = np.where(z > 0, np.log(np.maximum(z, np.finfo(e.dtype).tiny)) + mx, 0.0)
    lq = np.where(mask, logits - lse, NEG_INF_LOGIT)
    return q, lq


def decode(z_raw, z_mixed, z_target, mask, p, decoder, enc_dim, m, d_v, d_e, slope=0.2):
    """Logits of sampler.py:91-129."""
    B, _, d = z_raw.shape
    if decoder == "linear":
        return (z_mixed.reshape(B * m, d) @ p["sampler/w_linear"]).reshape(B, m)
    if decoder == "gat":
        zt = pad_target(z_target, enc_dim, m, d_v, d_e)
        W = p["sampler/W_gat"]
        pu = (z_raw.reshape(B * m, d) @ W).reshape(B, m, -1)
        pv = (zt @ W).reshape(B, 1, -1)
        da = W.shape[1]
        a = p["sampler/a_gat"]
        raw = (pu * a[:da, 0]).sum(axis=2) + (pv * a[da:, 0]).sum(axis=2)
        return leaky(raw, slope)
    if decoder == "gatv2":
        zt = pad_target(z_target, enc_dim, m, d_v, d_e)
        pair = np.concatenate([z_raw, np.broadcast_to(zt[:, None, :], (B, m, d))], axis=2).reshape(B * m, 2 * d)
        hidden = leaky(pair @ p["sampler/W_gatv2"], slope)
        return (hidden @ p["sampler/a_gatv2"]).reshape(B, m)
    if decoder == "trans":
        qt = z_target @ p["sampler/W_trans_target"]
        kn = (z_mixed.reshape(B * m, d) @ p["sampler/W_trans_nbr"]).reshape(B, m, -1)
        raw = (qt[:, None, :] * kn).sum(axis=2)
        counts = np.maximum(mask.sum(axis=1), 1).astype(np.float64)
        return raw * (1.0 / np.sqrt(counts))[:, None]
    raise ValueError(decoder)


def policy(ids, dts, mask, node_rows, edge_rows, tgt_rows, p, decoder, enc_dim, alpha, beta, d_v, d_e):
    """(q, log_q, z_raw, z_mixed, z_target) for one layer, float64."""
    B, m = ids.shape
    z_raw = encode_neighbors(ids, dts, mask, node_rows, edge_rows, p, enc_dim, alpha, beta)
    z_mixed = mixer(z_raw, mask, p)
    z_target = encode_target(tgt_rows, p, enc_dim, alpha, beta, B)
    logits = decode(z_raw, z_mixed, z_target, mask, p, decoder, enc_dim, m, d_v, d_e)
    q, lq = masked_softmax(logits, mask)
    return q, lq, z_raw, z_mixed, z_target


class OracleScorer:
    """Bound parameters + encoder constants; the interface OracleMiniBatch
    uses for adaptive layers."""

    def __init__(self, params, decoder, enc_dim, m, d_v, d_e, alpha, beta):
        self.p, self.decoder, self.enc_dim, self.m = params, decoder, enc_dim, m
        self.d_v, self.d_e, self.alpha, self.beta = d_v, d_e, alpha, beta

    def policy(self, nodes, ids, dts, mask, node_rows, edge_rows, tgt_rows):
        q, lq, *_ = policy(ids, dts, mask, node_rows, edge_rows, tgt_rows, self.p, self.decoder, self.enc_dim,
                           self.alpha, self.beta, self.d_v, self.d_e)
        return q, lq


def make_scorer(graph, cfg, seed):
    """The Trainer's sampler store + encoder config for `seed`
    (training.py:141-163) as an OracleScorer."""
    from .rng import derive_seed
    S_SAMPLER = 1
    span = cfg.time_span
    if span is None:
        span = float(graph.ts[-1] - graph.ts[0]) if graph.num_events > 1 else None
    alpha, beta = encoder_constants(cfg.enc_dim, span)
    p = sampler_params(derive_seed(seed, S_SAMPLER), cfg.enc_dim, cfg.m, graph.d_v, graph.d_e, cfg.decoder)
    return OracleScorer(p, cfg.decoder, cfg.enc_dim, cfg.m, graph.d_v, graph.d_e, alpha, beta)
