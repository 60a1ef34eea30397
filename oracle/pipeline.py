"""Mini-batch generation restated on the CPU (TEST INFRASTRUCTURE).

Follows the ★ lines of training.py: roots of an iteration (:364-382,
adaptive mini-batch selection off), ``_layer_neighborhoods`` (:232-292),
hop expansion (:301-314), ``_edge_feature_rows`` / ``_node_feature_rows``
(:207-230) and the PP slices (:316-345), with the cache of cache.py.  It is
both the parity oracle for end-to-end batches and the timed CPU baseline
(NF/FS phase timers like training.py:183).
"""

from __future__ import annotations

import time

import numpy as np

from . import finder as ofinder
from .cache import OracleCache
from .rng import S_FINDER, S_NEG, S_POLICY, derive_seed, substream


class OracleMiniBatch:
    def __init__(self, graph, cfg, seed=0, dtype=np.float64, scorer=None):
        self.g, self.cfg, self.seed, self.dtype = graph, cfg, int(seed), np.dtype(dtype)
        self.L = 2 if cfg.aggregator == "tgat" else 1
        self.budget = cfg.m if cfg.adaptive_neighbor else cfg.n
        E = graph.num_events
        window = cfg.window if cfg.window is not None else E
        start = E - window
        self.train_lo, self.train_hi = start, start + int(np.floor(cfg.split_ratios[0] * window))
        self.iters_per_epoch = int(np.ceil((self.train_hi - self.train_lo) / cfg.batch_size))
        self._dst_pool = None
        self.cache = None
        if graph.d_e and cfg.cache_fraction and cfg.cache_fraction > 0:
            self.cache = OracleCache(E, cfg.cache_fraction, epsilon=cfg.cache_epsilon, features=graph.edge_features)
        self.phase = {"NF": 0.0, "AS": 0.0, "FS": 0.0}
        if scorer is None and cfg.adaptive_neighbor:
            from .scoring import make_scorer
            scorer = make_scorer(graph, cfg, seed)
        self.scorer = scorer

    @property
    def dst_pool(self):
        if self._dst_pool is None:  # lazily: a full-size check feeds its own roots
            self._dst_pool = np.unique(self.g.dst[self.train_lo:self.train_hi])
        return self._dst_pool

    def roots_for_iteration(self, it):
        s = self.train_lo + (it % self.iters_per_epoch) * self.cfg.batch_size
        e = min(s + self.cfg.batch_size, self.train_hi)
        g = self.g
        rng = substream(self.seed, S_NEG, it)
        negs = self.dst_pool[rng.integers(0, self.dst_pool.size, size=e - s)]
        return (np.concatenate([g.src[s:e], g.dst[s:e], negs]).astype(np.int64),
                np.concatenate([g.ts[s:e]] * 3).astype(np.float64))

    # training.py:207-221
    def edge_rows(self, eids, mask, train_mode):
        g = self.g
        if not g.d_e:
            return None
        t0 = time.perf_counter()
        flat = eids[mask]
        if train_mode and self.cache is not None:
            feats, _ = self.cache.lookup(flat)
        else:
            feats = g.edge_features[flat]
        out = np.zeros(eids.shape + (g.d_e,), dtype=self.dtype)
        out[mask] = feats
        self.phase["FS"] += time.perf_counter() - t0
        return out

    # training.py:223-230
    def node_rows(self, ids, mask=None):
        g = self.g
        if not g.d_v:
            return None
        rows = g.node_features[ids].astype(self.dtype)
        if mask is not None:
            rows = rows * mask[..., None].astype(self.dtype)
        return rows

    # training.py:232-292
    def layer(self, nodes, times, layer, train_mode, it_key, rows=None):
        """rows: (split, base0, base1, B_global) global row keys of a root
        shard (None = the whole batch)."""
        g, cfg = self.g, self.cfg
        t0 = time.perf_counter()
        fseed = derive_seed(self.seed, S_FINDER, it_key, layer)
        split, base0, base1, B_global = rows if rows is not None else (None, 0, 0, None)
        idx, cnt = ofinder.batch_find_arrays(g, nodes, times, self.budget, policy=cfg.finder_policy, seed=fseed,
                                             row_base=base0, split=split, base1=base1)
        mask = np.arange(self.budget)[None, :] < cnt[:, None]
        safe = np.where(mask, idx, 0)
        ids = np.where(mask, g.tcsr_neighbors[safe], 0)
        tss = np.where(mask, g.tcsr_ts[safe], 0.0)
        eids = np.where(mask, g.tcsr_eids[safe], 0)
        dts = np.where(mask, times[:, None] - tss, 0.0)
        self.phase["NF"] += time.perf_counter() - t0
        rec = {"B": nodes.shape[0], "layer": layer, "idx": idx, "cnt": cnt, "ids": ids, "eids": eids, "dts": dts,
               "mask": mask, "tss": tss}
        if not cfg.adaptive_neighbor:
            rec.update(sel_ids=ids, sel_dts=dts, sel_eids=eids, sel_mask=mask)
            return rec
        B = nodes.shape[0]
        edge_rows = self.edge_rows(eids, mask, train_mode)
        node_rows = self.node_rows(ids, mask)
        if node_rows is not None:
            node_rows = node_rows.reshape(B, cfg.m, g.d_v)
        t0 = time.perf_counter()
        q, log_q = self.scorer.policy(nodes, ids, dts, mask, node_rows, edge_rows, self.node_rows(nodes))
        from .wor import sample_wor
        rng = substream(self.seed, S_POLICY, it_key, layer)
        grows = None
        if B_global is not None:
            i = np.arange(B)
            grows = np.where(i < split, base0 + i, base1 + (i - split))
        sel, smask, slq = sample_wor(q, log_q, cfg.n, rng, B_global=B_global, global_rows=grows)
        self.phase["AS"] += time.perf_counter() - t0
        safe_sel = np.maximum(sel, 0)
        r = np.arange(B)[:, None]
        rec.update(q=q, log_q=log_q, selected=sel, selected_mask=smask, selected_log_q=slq,
                   cand_edge_rows=edge_rows, cand_node_rows=node_rows,
                   sel_ids=np.where(smask, ids[r, safe_sel], 0), sel_dts=np.where(smask, dts[r, safe_sel], 0.0),
                   sel_eids=np.where(smask, eids[r, safe_sel], 0), sel_mask=smask)
        return rec

    # training.py:294-345 (mini-batch part: no aggregator compute)
    def generate(self, nodes, times, it_key, train_mode=True, layer_rows=None):
        """layer_rows: per layer (top first) (split, base0, base1, B_global)
        of a root shard, or None for the whole batch."""
        act = {self.L: (np.asarray(nodes, dtype=np.int64), np.asarray(times, dtype=np.float64))}
        recs = {}
        for l in range(self.L, 0, -1):
            tn, tt = act[l]
            rows = None if layer_rows is None else layer_rows[self.L - l]
            rec = self.layer(tn, tt, l, train_mode, it_key, rows=rows)
            recs[l] = rec
            if l > 1:
                w = rec["sel_ids"].shape[1]
                act[l - 1] = (np.concatenate([tn, rec["sel_ids"].ravel()]),
                              np.concatenate([tt, np.repeat(tt, w) - rec["sel_dts"].ravel()]))
                rec["next_v"], rec["next_t"] = act[l - 1]
        if self.cfg.aggregator == "graphmixer":
            rec = recs[1]
            rec["edge_rows"] = self.edge_rows(rec["sel_eids"], rec["sel_mask"], train_mode)
            rec["node_rows"] = self.node_rows(rec["sel_ids"], rec["sel_mask"])
        else:
            for l in range(1, self.L + 1):
                rec = recs[l]
                rec["edge_rows"] = self.edge_rows(rec["sel_eids"], rec["sel_mask"], train_mode)
                if l == 1:
                    rec["node_rows"] = self.node_rows(rec["sel_ids"], rec["sel_mask"])
                    rec["tgt_rows"] = self.node_rows(act[1][0])
        return [recs[l] for l in range(self.L, 0, -1)]

    def end_epoch(self):
        return None if self.cache is None else self.cache.maybe_replace()
