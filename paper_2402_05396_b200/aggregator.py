"""GraphMixer aggregator forward on the device.

The consumer of the mini-batch for GraphMixer models: training.py:318-330
turns layer 1's buffers (selected dts, mask, edge rows, node rows) into
messages (aggregators.py:58-71 ``build_messages``) and embeds every root
with ``graphmixer_layer`` (aggregators.py:140-145: mixer_forward, mixer.py
:31-51, then the mean over all slots, padding included).  The same mixer
machinery as K7 runs it (3xTF32 tcgen05 channel MLP in f32, FP64 GEMMs in
f64) with the model's own weights.

``model_params`` reproduces a fresh reference model store for these names
(init_time_encode_params aggregators.py:44-52, init_graphmixer_params
:135-137 -> init_mixer_params mixer.py:13-28, Glorot keyed by (seed, name)).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr
from .params import _glorot


def model_params(store_seed, n, d_v, d_e, d_time=100, time_span=None, prefix="model"):
    """name -> float64 array of a fresh reference model store (GraphMixer)."""
    span = float(time_span) if time_span else float(d_time)
    span = max(span, 2.0)
    p = {f"{prefix}/time_w": span ** (-np.arange(d_time, dtype=np.float64) / max(d_time - 1, 1)),
         f"{prefix}/time_b": np.zeros(d_time)}
    d = d_v + d_e + d_time
    pre = f"{prefix}/gmixer"
    for ln in ("ln1", "ln2"):
        p[f"{pre}/{ln}_gamma"] = np.ones(d)
        p[f"{pre}/{ln}_beta"] = np.zeros(d)
    p[f"{pre}/Wc1"] = _glorot(store_seed, f"{pre}/Wc1", (d, d))
    p[f"{pre}/bc1"] = np.zeros(d)
    p[f"{pre}/Wc2"] = _glorot(store_seed, f"{pre}/Wc2", (d, d))
    p[f"{pre}/bc2"] = np.zeros(d)
    p[f"{pre}/Wt1"] = _glorot(store_seed, f"{pre}/Wt1", (n, n))
    p[f"{pre}/bt1"] = np.zeros(n)
    p[f"{pre}/Wt2"] = _glorot(store_seed, f"{pre}/Wt2", (n, n))
    p[f"{pre}/bt2"] = np.zeros(n)
    return p


class GraphMixerAggregator:
    """Device GraphMixer layer for slot count n (RunConfig.n)."""

    _NAMES = (("time_w", "time_w"), ("time_b", "time_b"), ("ln1_g", "gmixer/ln1_gamma"),
              ("ln1_b", "gmixer/ln1_beta"), ("Wc1", "gmixer/Wc1"), ("bc1", "gmixer/bc1"), ("Wc2", "gmixer/Wc2"),
              ("bc2", "gmixer/bc2"), ("ln2_g", "gmixer/ln2_gamma"), ("ln2_b", "gmixer/ln2_beta"),
              ("Wt1", "gmixer/Wt1"), ("bt1", "gmixer/bt1"), ("Wt2", "gmixer/Wt2"), ("bt2", "gmixer/bt2"))

    def __init__(self, params, n, d_v, d_e, d_time=100, precision="float64", device=None, prefix="model",
                 tensor_cores=True):
        t = _lib.torch()
        _lib.require_cuda("the GraphMixer aggregator")
        if precision not in ("float64", "float32"):
            raise ValueError(f"unknown precision {precision!r}")
        self.n, self.d_v, self.d_e, self.d_time = int(n), int(d_v), int(d_e), int(d_time)
        self.d_msg = self.d_v + self.d_e + self.d_time
        self.precision = precision
        self.dtype = t.float64 if precision == "float64" else t.float32
        dev = device if device is not None else t.device("cuda", t.cuda.current_device())
        self.dev = dev
        self._t = {}
        for field, name in self._NAMES:
            self._t[field] = t.as_tensor(np.ascontiguousarray(params[f"{prefix}/{name}"])).to(dev, self.dtype)
        self.c = _lib.tg_gmixer_model(1 if precision == "float64" else 0, self.n, self.d_v, self.d_e, self.d_time,
                                      0 if tensor_cores else 1, *[ptr(self._t[f]) for f, _ in self._NAMES])
        self._ws = None

    def workspace(self, B):
        sz = _lib.ctypes.c_size_t(0)
        check(_lib.lib.tg_graphmixer_workspace(self.c, int(B), _lib.ctypes.byref(sz)))
        if self._ws is None or self._ws.numel() < sz.value:
            t = _lib.torch()
            self._ws = t.empty(max(int(sz.value), 1), dtype=t.uint8, device=self.dev)
        return self._ws

    def forward(self, dts, mask, edge_rows=None, node_rows=None, out=None, stream=None):
        """h [B, d_msg] from one layer's buffers (the generator's ``sel_dts``,
        ``sel_mask``, ``edge_rows``, ``node_rows``; rows may be pitched views)."""
        t = _lib.torch()
        B, n = int(dts.shape[0]), int(dts.shape[1])
        if n != self.n:
            raise ValueError(f"model built for {self.n} slots, got {n}")

        def rows(x, d):
            if not d:
                return None, 0
            if x is None:
                raise ValueError("feature rows required")
            if x.dtype != t.float32 or x.stride(-1) != 1:
                raise ValueError("feature rows must be f32 with contiguous rows")
            return x, int(x.stride(-2))

        er, eld = rows(edge_rows, self.d_e)
        nr, nld = rows(node_rows, self.d_v)
        dt = dts.contiguous() if dts.dtype == t.float64 else dts.to(t.float64).contiguous()
        mk = mask.contiguous().view(t.uint8) if mask.dtype == t.bool else mask.to(t.uint8).contiguous()
        if out is None:
            out = t.empty((B, self.d_msg), dtype=self.dtype, device=self.dev)
        ws = self.workspace(B)
        check(_lib.lib.tg_graphmixer_forward(self.c, ptr(nr), nld, ptr(er), eld, ptr(dt), ptr(mk), B, ptr(out),
                                             int(out.stride(0)), ptr(ws), int(ws.numel()), stream_ptr(stream)))
        return out

    def forward_record(self, rec, stream=None):
        """h of a MiniBatchGenerator layer record (training.py:318-330)."""
        return self.forward(rec["sel_dts"], rec["sel_mask"], rec.get("edge_rows"), rec.get("node_rows"),
                            stream=stream)


# ---------------------------------------------------------------------------
# TGAT (aggregators.py:74-132): two attention layers, bottom-up
# ---------------------------------------------------------------------------

def tgat_params(store_seed, d_v, d_e, hidden=100, d_time=100, layers=2, time_span=None, prefix="model"):
    """name -> float64 array of a fresh reference TGAT model store
    (training.py:187-198: init_time_encode_params + init_tgat_params per layer)."""
    span = float(time_span) if time_span else float(d_time)
    span = max(span, 2.0)
    p = {f"{prefix}/time_w": span ** (-np.arange(d_time, dtype=np.float64) / max(d_time - 1, 1)),
         f"{prefix}/time_b": np.zeros(d_time)}
    for layer in range(1, layers + 1):
        d_in = d_v if layer == 1 else hidden
        d_msg = d_in + d_e + d_time
        pre = f"{prefix}/tgat{layer}"
        p[f"{pre}/W_q"] = _glorot(store_seed, f"{pre}/W_q", (d_in + d_time, hidden))
        p[f"{pre}/b_s"] = np.zeros(hidden)
        p[f"{pre}/W_k"] = _glorot(store_seed, f"{pre}/W_k", (d_msg, hidden))
        p[f"{pre}/b_k"] = np.zeros(hidden)
        p[f"{pre}/W_v"] = _glorot(store_seed, f"{pre}/W_v", (d_msg, hidden))
        p[f"{pre}/b_v"] = np.zeros(hidden)
    return p


class TGATModel:
    """Device TGAT aggregator (ModelConfig aggregator='tgat')."""

    def __init__(self, params, d_v, d_e, hidden=100, d_time=100, layers=2, slots=10, precision="float64",
                 device=None, prefix="model", tensor_cores=False):
        # f32 projections default to FFMA: the bilinear attention scores q.K
        # amplify the 3xTF32 GEMM error past 1e-5 (as K7's trans decoder)
        t = _lib.torch()
        _lib.require_cuda("the TGAT aggregator")
        if precision not in ("float64", "float32"):
            raise ValueError(f"unknown precision {precision!r}")
        self.d_v, self.d_e, self.hidden, self.d_time = int(d_v), int(d_e), int(hidden), int(d_time)
        self.layers, self.slots = int(layers), int(slots)
        self.dtype = t.float64 if precision == "float64" else t.float32
        self.dev = device if device is not None else t.device("cuda", t.cuda.current_device())
        up = lambda name: t.as_tensor(np.ascontiguousarray(params[f"{prefix}/{name}"])).to(self.dev, self.dtype)  # noqa: E731
        self._keep = {"time_w": up("time_w"), "time_b": up("time_b")}
        self.c = {}
        for layer in range(1, self.layers + 1):
            pre = f"tgat{layer}"
            ts = {k: up(f"{pre}/{k}") for k in ("W_q", "b_s", "W_k", "b_k", "W_v", "b_v")}
            self._keep[layer] = ts
            d_in = self.d_v if layer == 1 else self.hidden
            self.c[layer] = _lib.tg_tgat_layer(
                1 if precision == "float64" else 0, 0 if tensor_cores else 1, d_in, self.d_e, self.d_time,
                self.hidden, self.slots, ptr(self._keep["time_w"]), ptr(self._keep["time_b"]),
                *[ptr(ts[k]) for k in ("W_q", "b_s", "W_k", "b_k", "W_v", "b_v")])
        self._ws = None

    def _workspace(self, layer, B):
        sz = _lib.ctypes.c_size_t(0)
        check(_lib.lib.tg_tgat_workspace(self.c[layer], int(B), _lib.ctypes.byref(sz)))
        if self._ws is None or self._ws.numel() < sz.value:
            t = _lib.torch()
            self._ws = t.empty(max(int(sz.value), 1), dtype=t.uint8, device=self.dev)
        return self._ws

    def layer(self, layer, h_tgt, h_nbr, edge_rows, dts, mask, stream=None):
        """(h [B, hidden], tau [B, s]) of tgat_layer(layer) (aggregators.py:74-132).
        h_tgt [B, d_in], h_nbr [B*s, d_in]: f32 feature rows (layer 1) or
        the previous layer's h; edge_rows [B*s, d_e] f32 (pitched views ok)."""
        t = _lib.torch()
        B = int(dts.shape[0])
        if int(dts.shape[1]) != self.slots:
            raise ValueError(f"model built for {self.slots} slots, got {int(dts.shape[1])}")

        def arg(x):
            if x is None or x.numel() == 0:
                return None, 0, 0
            if x.stride(-1) != 1:
                raise ValueError("rows must be contiguous")
            if x.dtype not in (t.float32, self.dtype):
                raise ValueError(f"embeddings must be f32 feature rows or {self.dtype}")
            return x, int(x.stride(-2)), 1 if x.dtype == t.float32 else 0

        ht, tld, tf = arg(h_tgt)
        hn, nld, nf = arg(h_nbr)
        er = edge_rows if self.d_e else None
        eld = int(er.stride(-2)) if er is not None else 0
        dt = dts.contiguous() if dts.dtype == t.float64 else dts.to(t.float64).contiguous()
        mk = mask.contiguous().view(t.uint8) if mask.dtype == t.bool else mask.to(t.uint8).contiguous()
        h = t.empty((B, self.hidden), dtype=self.dtype, device=self.dev)
        tau = t.empty((B, self.slots), dtype=self.dtype, device=self.dev)
        ws = self._workspace(layer, B)
        check(_lib.lib.tg_tgat_forward(self.c[layer], ptr(ht), tld, tf, ptr(hn), nld, nf, ptr(er), eld, ptr(dt),
                                       ptr(mk), B, ptr(h), int(h.stride(0)), ptr(tau), ptr(ws), int(ws.numel()),
                                       stream_ptr(stream)))
        return h, tau

    def forward_records(self, recs, stream=None):
        """h of the roots from a 2-layer MiniBatchGenerator batch (records
        layer L first), bottom-up as training.py:333-356."""
        by = {r["layer"]: r for r in recs}
        h = None
        for layer in range(1, self.layers + 1):
            rec = by[layer]
            B = int(rec["sel_dts"].shape[0])
            if layer == 1:
                h_nbr = rec.get("node_rows")
                h_tgt = rec.get("tgt_rows")
                if h_nbr is not None:
                    h_nbr = h_nbr.reshape(-1, h_nbr.shape[-1])
            else:
                h_tgt, h_nbr = h[:B], h[B:]
            er = rec.get("edge_rows")
            if er is not None:
                er = er.reshape(-1, er.shape[-1])
            h, tau = self.layer(layer, h_tgt, h_nbr, er, rec["sel_dts"], rec["sel_mask"], stream=stream)
            rec["h"], rec["tau"] = h, tau
        return h
