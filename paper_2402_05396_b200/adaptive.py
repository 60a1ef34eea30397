"""Adaptive layers of the mini-batch pipeline (training.py:255-292).

Per layer: candidates (K2 with budget m, fused with the candidate edge-row
slice through the cache, training.py:264), candidate node rows and the
roots' node rows (training.py:265-267, 273), K7 scoring -> (q, log q), K8
sampling without replacement with the policy substream
(training.py:277-278), then the selection gather + hop expansion
(training.py:281-291, 311-314) and the PP edge rows of the selection
(training.py:320 / 339).
"""

from __future__ import annotations

from . import _lib
from ._lib import check, ptr
from .finder import find_args
from .graph import feat_store, padded_rows, row_pitch
from .params import ScoringModel, encoder_constants, sampler_params
from .sampler import sample_wor_device
from .scoring import score_policy
from .seeds import S_POLICY, S_SAMPLER, derive_seed, substream


class AdaptiveLayer:
    def __init__(self, gen, params=None):
        g, cfg = gen.graph, gen.cfg
        self.gen = gen
        span = cfg.time_span
        if span is None:
            ts = g.ts
            span = float((ts[-1] - ts[0]).item()) if g.num_events > 1 else None
        alpha, beta = encoder_constants(cfg.enc_dim, span)
        if params is None:
            params = sampler_params(derive_seed(gen.seed, S_SAMPLER), cfg.enc_dim, cfg.m, g.d_v, g.d_e, cfg.decoder)
        self.params = params
        self.model = ScoringModel(params, cfg.decoder, cfg.enc_dim, cfg.m, g.d_v, g.d_e, alpha, beta,
                                  precision=cfg.precision, device=g.device)

    def allocate(self, ws):
        t = _lib.torch()
        g, cfg, dev = self.gen.graph, self.gen.cfg, self.gen.dev
        m, n = cfg.m, cfg.n
        dt = self.model.dtype
        for rec in ws.layers:
            B = rec["B"]
            if g.d_e:
                rec["cand_edge_rows"] = padded_rows((B, m), g.d_e, dev, zero=False)
            if g.d_v:
                rec["cand_node_rows"] = padded_rows((B, m), g.d_v, dev, zero=False)
                if cfg.decoder != "linear":
                    rec["root_rows"] = padded_rows((B,), g.d_v, dev, zero=False)
            rec["q"] = t.empty((B, m), dtype=dt, device=dev)
            rec["log_q"] = t.empty((B, m), dtype=dt, device=dev)
            rec["selected"] = t.empty((B, n), dtype=t.int64, device=dev)
            rec["selected_mask"] = t.empty((B, n), dtype=t.bool, device=dev)
            rec["selected_log_q"] = t.empty((B, n), dtype=dt, device=dev)
            rec["sel_ids"] = t.empty((B, n), dtype=t.int64, device=dev)
            rec["sel_eids"] = t.empty((B, n), dtype=t.int64, device=dev)
            rec["sel_dts"] = t.empty((B, n), dtype=t.float64, device=dev)

    def run_layer(self, rec, qv, qt, it_key, l, seed, train_mode, ws, st, rows=None, B_global=None,
                  stores=None, stream=None):
        if stream is None:
            stream = _lib.torch().cuda.current_stream()
        """st: the launching stream as a C pointer; stream: the same as a
        torch stream (None = current)."""
        gen = self.gen
        g, cfg = gen.graph, gen.cfg
        cache = gen.cache if train_mode else None
        estore, nstore = stores if stores is not None else (gen.edge_store(), feat_store(g.node_features))
        ccache = cache.c_cache() if cache is not None else None
        B = rec["B"]
        # candidates + their edge rows through the cache (training.py:241-264)
        a = find_args(qv, qt, cfg.m, gen.policy, seed, rows=rows, ids=rec["ids"], eids=rec["eids"], dts=rec["dts"],
                      mask=rec["mask"], feat_out=rec.get("cand_edge_rows"))
        if a.feat_out:
            a.feat_ld = int(rec["cand_edge_rows"].stride(-2))
        check(_lib.lib.tg_find(g.c_graph(), a, estore, ccache, st))
        if g.d_v:  # node rows * mask (signed zeros, training.py:227-229)
            check(_lib.lib.tg_lookup_gather(ptr(rec["ids"]), ptr(rec["mask"]), B * cfg.m, nstore, None, 1,
                                            ptr(rec["cand_node_rows"]), row_pitch(g.d_v), st))
            if "root_rows" in rec:
                check(_lib.lib.tg_lookup_gather(ptr(qv), None, B, nstore, None, 0, ptr(rec["root_rows"]), row_pitch(g.d_v),
                                                st))
        # K7 (training.py:269-276); optional CUDA events around it (bench.py)
        ev = rec.get("score_events")
        if ev is not None:
            ev[0].record(stream)
        score_policy(self.model, rec["ids"], rec["dts"], rec["mask"], rec.get("cand_node_rows"),
                     rec.get("cand_edge_rows"), rec.get("root_rows"), q=rec["q"], log_q=rec["log_q"],
                     stream=stream)
        if ev is not None:
            ev[1].record(stream)
        # K8 with the policy substream (training.py:277-278)
        rng = substream(gen.seed, S_POLICY, it_key, l)
        sample_wor_device(rec["q"], rec["log_q"], cfg.n, rng, B_global=B_global, rows=rows,
                          selected=rec["selected"], sel_mask=rec["selected_mask"], sel_log_q=rec["selected_log_q"],
                          stream=stream)
        # selection gather + next-hop queries (training.py:281-291, 311-314)
        check(_lib.lib.tg_select_expand(ptr(rec["ids"]), ptr(rec["eids"]), ptr(rec["dts"]), ptr(rec["selected"]),
                                        ptr(rec["selected_mask"]), ptr(qv), ptr(qt), B, cfg.m, cfg.n,
                                        ptr(rec["sel_ids"]), ptr(rec["sel_eids"]), ptr(rec["sel_dts"]),
                                        ptr(rec.get("next_v")), ptr(rec.get("next_t")), st))
        rec["sel_mask"] = rec["selected_mask"]
        # PP edge rows of the selection through the cache (training.py:320 / 339)
        if "edge_rows" in rec:
            check(_lib.lib.tg_lookup_gather(ptr(rec["sel_eids"]), ptr(rec["sel_mask"]), B * cfg.n, estore, ccache, 0,
                                            ptr(rec["edge_rows"]), row_pitch(g.d_e), st))
