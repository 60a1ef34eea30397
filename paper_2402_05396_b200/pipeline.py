"""Mini-batch generation: the Trainer's NF -> (AS) -> FS path on the device.

Mirrors the hot path of training.py (the Trainer is OUT of scope; this is the
part of it SURVEY §8 marks ★):

  * roots of iteration ``it`` (training.py:364-382): a chronological slice of
    the training split, negatives from ``substream(seed, S_NEG, it)``;
  * per layer l = L..1 ``_layer_neighborhoods`` (training.py:232-292): finder
    seed ``derive_seed(seed, S_FINDER, it, l)``, materialised ids/dts/eids/mask;
  * hop expansion (training.py:307-314): next queries [targets || children];
  * the PP feature slices (training.py:316-345): edge rows of every layer's
    selection through the cache in train mode, node rows where the
    aggregator reads them.

Non-adaptive layers are ONE kernel launch each (K2 fused with K3 and K4/K5).
Adaptive layers (candidates -> score -> sample) live in ``adaptive.py``.
Output buffers are persistent (allocated once per root count) so a step can
be replayed from a CUDA graph; the tensors returned by ``generate`` are valid
until the next call.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import TG_RECENT, TG_UNIFORM, check, ptr, stream_ptr
from .cache import make_cache
from .finder import find_args
from .graph import feat_store, padded_rows, row_pitch
from .seeds import S_BATCH, S_FINDER, S_NEG, derive_seed, substream


@dataclass
class PathConfig:
    """The RunConfig fields (training.py:47-108) that drive the hot path."""

    aggregator: str = "graphmixer"
    decoder: str = None
    finder_policy: str = None
    m: int = 25
    n: int = 10
    batch_size: int = 600
    cache_fraction: float = 0.2
    cache_epsilon: float = None
    adaptive_neighbor: bool = True
    enc_dim: int = 100
    split_ratios: tuple = (0.6, 0.2, 0.2)
    window: int = None
    time_span: float = None
    hot_tier: bool = False
    precision: str = "float64"   # sampler compute dtype (RunConfig.precision, training.py:75)
    adaptive_minibatch: bool = False  # importance-weighted batch selection (RunConfig, training.py:364-367)
    gamma: float = 0.1                # selector floor (init_scores gamma, selector.py:36)

    def __post_init__(self):
        if self.aggregator not in ("tgat", "graphmixer"):
            raise ValueError(f"unknown aggregator {self.aggregator!r}")
        if self.decoder is None:
            self.decoder = "gatv2" if self.aggregator == "tgat" else "linear"
        if self.finder_policy is None:
            self.finder_policy = "uniform" if self.aggregator == "tgat" else "recent"
        if self.finder_policy not in ("uniform", "recent"):
            raise ValueError(f"unknown finder policy {self.finder_policy!r}")
        if not (1 <= self.n <= self.m):
            raise ValueError(f"need 1 <= n <= m, got n={self.n}, m={self.m}")
        if self.precision not in ("float64", "float32"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.decoder not in ("linear", "gat", "gatv2", "trans"):
            raise ValueError(f"unknown decoder {self.decoder!r}")

    @property
    def layers(self):
        return 2 if self.aggregator == "tgat" else 1

    @property
    def budget(self):
        return self.m if self.adaptive_neighbor else self.n


def train_range(num_events, ratios=(0.6, 0.2, 0.2), window=None):
    """Training eid range of chronological_split (graph.py:274-289)."""
    if window is None:
        window = num_events
    start = num_events - window
    b1 = start + int(np.floor(ratios[0] * window))
    return start, b1


@dataclass
class Workspace:
    """Persistent per-layer output buffers for R1 roots."""

    R1: int
    layers: list = field(default_factory=list)
    roots_v: object = None
    roots_t: object = None
    valid: object = None


class MiniBatchGenerator:
    """Device mini-batch generation for one seed (Trainer state subset)."""

    def __init__(self, graph, cfg, seed=0, cache=None, stream=None):
        t = _lib.torch()
        self.graph, self.cfg, self.seed = graph, cfg, int(seed)
        self.L = cfg.layers
        self.budget = cfg.budget
        self.policy = TG_UNIFORM if cfg.finder_policy == "uniform" else TG_RECENT
        self.dev = graph.device
        if cache is None and graph.d_e and cfg.cache_fraction and cfg.cache_fraction > 0:
            # a sharded table (placement.py) always serves resident rows from a
            # local hot tier; misses go to the owner shard over NVLink
            sharded = hasattr(graph.edge_features, "c_store")
            cache = make_cache(graph.num_events, cfg.cache_fraction, epsilon=cfg.cache_epsilon,
                               features=graph.edge_features, hot_tier=cfg.hot_tier or sharded)
        self.cache = cache
        lo, hi = train_range(graph.num_events, cfg.split_ratios, cfg.window)
        self.train_lo, self.train_hi = lo, hi
        if hi <= lo:
            raise ValueError("empty training split")
        self.iters_per_epoch = int(np.ceil((hi - lo) / cfg.batch_size))
        self._dst_pool = None
        self._ws = {}
        self.stream = stream
        self._adaptive = None
        self.scores = None
        if cfg.adaptive_minibatch:
            from .selector import init_scores
            self.scores = init_scores(hi - lo, gamma=cfg.gamma, base_eid=lo)
        self._side = {}
        self._slot_streams = {}
        self.merge_gathers = True  # non-adaptive: every layer's edge rows in one K5 launch (generate())
        if cfg.adaptive_neighbor:
            from .adaptive import AdaptiveLayer
            self._adaptive = AdaptiveLayer(self)

    def edge_store(self):
        """Edge-row source: the cache's hot tier when it has one, else the table."""
        g = self.graph
        if not g.d_e:
            return None
        if self.cache is not None and self.cache.hot is not None:
            return self.cache.c_store()
        return feat_store(g.edge_features)

    # -- roots ---------------------------------------------------------------
    def dst_pool(self):
        if self._dst_pool is None:
            t = _lib.torch()
            self._dst_pool = t.unique(self.graph.dst[self.train_lo:self.train_hi]).cpu().numpy()
        return self._dst_pool

    def roots_for_iteration(self, it):
        """(nodes int64[3b], times f64[3b]) as numpy, like train_iteration
        (training.py:375-382) with adaptive_minibatch off."""
        b_start = self.train_lo + (it % self.iters_per_epoch) * self.cfg.batch_size
        b_end = min(b_start + self.cfg.batch_size, self.train_hi)
        src = self.graph.src[b_start:b_end].cpu().numpy()
        dst = self.graph.dst[b_start:b_end].cpu().numpy()
        ts = self.graph.ts[b_start:b_end].cpu().numpy()
        b = src.shape[0]
        pool = self.dst_pool()
        rng = substream(self.seed, S_NEG, it)
        negs = pool[rng.integers(0, pool.size, size=b)]
        return np.concatenate([src, dst, negs]).astype(np.int64), np.concatenate([ts, ts, ts]).astype(np.float64)

    def select_roots(self, it):
        """Device roots of iteration ``it`` with adaptive mini-batch selection
        (training.py:364-382): K9 draws the batch's training eids from the
        importance scores with substream(seed, S_BATCH, it), positives are
        gathered on the device, negatives come from substream(seed, S_NEG, it).
        Returns (nodes, times, eids) as CUDA tensors."""
        t = _lib.torch()
        from .selector import select_batch
        if self.scores is None:
            raise ValueError("select_roots needs PathConfig(adaptive_minibatch=True)")
        b = min(self.cfg.batch_size, self.scores.num_edges)
        eids = select_batch(self.scores, b, substream(self.seed, S_BATCH, it))
        g = self.graph
        pool = self.dst_pool()
        rng = substream(self.seed, S_NEG, it)
        negs = t.as_tensor(pool[rng.integers(0, pool.size, size=b)]).to(eids.device)
        nodes = t.cat([g.src[eids], g.dst[eids], negs])
        ts = g.ts[eids]
        return nodes, t.cat([ts, ts, ts]), eids

    def update_scores(self, eids, pos_logits):
        """Eq. 10 after the model's forward pass (training.py:403-404)."""
        from .selector import update_scores
        return update_scores(self.scores, eids, pos_logits)

    # -- buffers -------------------------------------------------------------
    def workspace(self, R1, slot=0):
        ws = self._ws.get((R1, slot))
        if ws is not None:
            return ws
        t = _lib.torch()
        dev, w, g = self.dev, self.budget, self.graph
        ws = Workspace(R1=R1)
        ws.roots_v = t.empty(R1, dtype=t.int64, device=dev)
        ws.roots_t = t.empty(R1, dtype=t.float64, device=dev)
        ws.valid = t.zeros(1, dtype=t.int64, device=dev)
        B = R1
        sel_w = self.cfg.n if self.cfg.adaptive_neighbor else w
        for l in range(self.L, 0, -1):
            rec = {"B": B, "layer": l}
            rec["ids"] = t.empty((B, w), dtype=t.int64, device=dev)
            rec["eids"] = t.empty((B, w), dtype=t.int64, device=dev)
            rec["dts"] = t.empty((B, w), dtype=t.float64, device=dev)
            rec["mask"] = t.empty((B, w), dtype=t.bool, device=dev)
            if l > 1:
                rec["next_v"] = t.empty(B * (1 + sel_w), dtype=t.int64, device=dev)
                rec["next_t"] = t.empty(B * (1 + sel_w), dtype=t.float64, device=dev)
            if g.d_e:
                rec["edge_rows"] = padded_rows((B, sel_w), g.d_e, dev, zero=False)
            if g.d_v and (self.cfg.aggregator == "graphmixer" or l == 1):
                rec["node_rows"] = padded_rows((B, sel_w), g.d_v, dev, zero=False)
                if self.cfg.aggregator == "tgat":
                    rec["tgt_rows"] = padded_rows((B,), g.d_v, dev, zero=False)
            ws.layers.append(rec)
            B = B * (1 + sel_w)
        if self._adaptive is not None:
            self._adaptive.allocate(ws)
        self._ws[(R1, slot)] = ws
        return ws

    # -- the hot path ----------------------------------------------------------
    def seeds_for(self, it_key):
        return {l: derive_seed(self.seed, S_FINDER, it_key, l) for l in range(1, self.L + 1)}

    def slot_stream(self, slot):
        """Stream of in-flight slot `slot` (0: the generator's / current stream)."""
        t = _lib.torch()
        if slot == 0:
            return self.stream if self.stream is not None else t.cuda.current_stream()
        if slot not in self._slot_streams:
            self._slot_streams[slot] = t.cuda.Stream(device=self.dev)
        return self._slot_streams[slot]

    def generate(self, nodes, times, it_key, train_mode=True, finder_seeds=None, layer_rows=None, events=None,
                 overlap=True, slot=0, seed_dev=None, stream=None):
        """Records for layers L..1 (list, layer L first) for device roots.

        nodes/times: int64/f64 CUDA tensors (R1,).  The returned dicts hold
        ``sel_ids, sel_dts, sel_eids, sel_mask`` and the feature rows.
        layer_rows: per-layer shard.LayerRows (top first) when these roots
        are one rank's block of a root-sharded batch (global RNG keys).
        overlap: the row slices of a layer (K5) run on a side stream,
        overlapping the next layer's finder; the call joins it before
        returning, so outputs are ordered on the caller's stream.
        events: optional list of (start, end, mid) CUDA events, one triple per
        layer: start/end around the layer's launches, mid after the finder
        (per-kernel timing in bench.py; forces overlap off).
        slot: batches in flight.  Slot k has its own output buffers and
        stream (``slot_stream(k)``), so a data loader can generate batch
        i+1 while batch i is consumed; outputs of slot k stay valid until
        the next call with slot k.  Cache counting commutes, so results are
        identical to the sequential order.  A slot's stream first waits for
        the caller's current stream, so roots produced there (select_roots,
        index ops) are complete before the finder reads them; consumers
        wait on ``slot_stream(k)`` (or ``join``) before reading the outputs.
        Slot 0 IS the caller's stream (outputs ordered like any op), so a
        loader keeping several batches in flight uses slots 1..K: a batch
        on slot 0 would make every later slot wait for it.
        """
        g = self.graph
        R1 = int(nodes.shape[0])
        ws = self.workspace(R1, slot)
        seeds = finder_seeds if finder_seeds is not None else (self.seeds_for(it_key) if seed_dev is None else None)
        if stream is not None:
            cur = stream
        else:
            cur = self.slot_stream(slot)
            caller = _lib.torch().cuda.current_stream(self.dev)
            if cur != caller:
                cur.wait_stream(caller)
        st = stream_ptr(cur)
        cgraph = g.c_graph()
        estore = self.edge_store()
        use_cache = train_mode and self.cache is not None
        ccache = self.cache.c_cache() if use_cache else None
        qv, qt = nodes, times
        out = []
        t = _lib.torch()
        side = None
        # non-adaptive layers: the edge-row slices of every layer go out as
        # ONE K5 launch after the last finder (tg_gather_rows_multi) -- a
        # per-layer launch of the small hop-1 slice competed with the big one
        # for SM slots and ran at a third of its speed with batches in flight
        merge = self._adaptive is None and "edge_rows" in ws.layers[0] and self.merge_gathers
        segs = []
        if overlap and events is None and self.L > 1 and not merge:
            if slot not in self._side:
                self._side[slot] = t.cuda.Stream(device=self.dev)
            side = self._side[slot]
        for li, rec in enumerate(ws.layers):
            l = rec["layer"]
            lr = layer_rows[li] if layer_rows is not None else None
            rows = lr.c_rowmap() if lr is not None else None
            if events is not None:
                events[li][0].record(cur)
            if self._adaptive is not None:
                if seed_dev is not None:
                    raise ValueError("seed_dev (graph replay) covers non-adaptive layers only")
                self._adaptive.run_layer(rec, qv, qt, it_key, l, seeds[l], train_mode, ws, st, rows=rows,
                                         B_global=lr.B_global if lr is not None else None,
                                         stores=(estore, feat_store(g.node_features)), stream=cur)
                if events is not None:
                    events[li][2].record(cur)
                self._node_rows(rec, qv, st)
            else:
                # K2+K3: find + materialise + expand, cache accounting of the
                # selected rows (training.py:241-253, 311-314; cache.py:78-82)
                a = find_args(qv, qt, self.budget, self.policy, seeds[l] if seed_dev is None else 0, rows=rows,
                              seed_ptr=seed_dev[li] if seed_dev is not None else None,
                              ids=rec["ids"], eids=rec["eids"], dts=rec["dts"], mask=rec["mask"],
                              next_v=rec.get("next_v"), next_t=rec.get("next_t"), valid_count=ws.valid)
                check(_lib.lib.tg_find(cgraph, a, None, ccache, st))
                if events is not None:
                    events[li][2].record(cur)
                rec["sel_ids"], rec["sel_eids"] = rec["ids"], rec["eids"]
                rec["sel_dts"], rec["sel_mask"] = rec["dts"], rec["mask"]
                gst = st
                if side is not None and l > 1:
                    side.wait_stream(cur)
                    gst = stream_ptr(side)
                # K5: the layer's edge rows (training.py:207-221), routed through the hot tier
                if "edge_rows" in rec and merge:
                    segs.append((rec["eids"], rec["mask"], rec["B"] * self.budget, rec["edge_rows"]))
                elif "edge_rows" in rec:
                    check(_lib.lib.tg_gather_rows(ptr(rec["eids"]), ptr(rec["mask"]), rec["B"] * self.budget, estore,
                                                  ptr(self.cache.slot_of) if self.cache is not None else None, 0,
                                                  ptr(rec["edge_rows"]), row_pitch(g.d_e), gst))
                self._node_rows(rec, qv, gst)
            if merge and li == len(ws.layers) - 1 and segs:
                arr = (_lib.tg_gather_seg * len(segs))(*[_lib.tg_gather_seg(ptr(e), ptr(mk), n, ptr(o))
                                                         for e, mk, n, o in segs])
                check(_lib.lib.tg_gather_rows_multi(arr, len(segs), estore,
                                                    ptr(self.cache.slot_of) if self.cache is not None else None, 0,
                                                    row_pitch(g.d_e), st))
            if events is not None:
                events[li][1].record(cur)
            rec["queries"] = (qv, qt)
            out.append(rec)
            if l > 1:
                qv, qt = rec["next_v"], rec["next_t"]
        if side is not None:
            cur.wait_stream(side)
        return out

    def generate_batched(self, batches, train_mode=True, layer_rows=None, stream=None):
        """Several non-adaptive mini-batches at once, layer by layer: ONE
        finder launch per layer for all of them (tg_find_batch) and ONE K5
        launch for every layer's rows (tg_gather_rows_multi), instead of a
        chain of small launches per batch -- what a root shard's 1/N batches
        need to keep the GPU busy.  ``batches``: list of (nodes, times,
        seed_dev, slot) -- seed_dev the per-layer u64 finder seeds on the
        device (layer L first), slot the workspace key.  Results are
        bit-identical to ``generate`` per batch.  Runs on ``stream`` (default:
        current); returns one record list per batch."""
        if self._adaptive is not None:
            raise ValueError("generate_batched covers non-adaptive layers")
        t = _lib.torch()
        g = self.graph
        cur = stream if stream is not None else t.cuda.current_stream(self.dev)
        st = stream_ptr(cur)
        cgraph = g.c_graph()
        estore = self.edge_store()
        ccache = self.cache.c_cache() if (train_mode and self.cache is not None) else None
        wss = [self.workspace(int(nodes.shape[0]), slot) for nodes, _, _, slot in batches]
        qs = [(nodes, times) for nodes, times, _, _ in batches]
        outs = [[] for _ in batches]
        segs = []
        for li in range(self.L):
            lr = layer_rows[li] if layer_rows is not None else None
            rows = lr.c_rowmap() if lr is not None else None
            args = []
            for b, (ws, (qv, qt)) in enumerate(zip(wss, qs)):
                rec = ws.layers[li]
                args.append(find_args(qv, qt, self.budget, self.policy, 0, rows=rows, seed_ptr=batches[b][2][li],
                                      ids=rec["ids"], eids=rec["eids"], dts=rec["dts"], mask=rec["mask"],
                                      next_v=rec.get("next_v"), next_t=rec.get("next_t"), valid_count=ws.valid))
            arr = (_lib.tg_find_args * len(args))(*args)
            check(_lib.lib.tg_find_batch(cgraph, arr, len(args), ccache, st))
            for b, (ws, (qv, qt)) in enumerate(zip(wss, qs)):
                rec = ws.layers[li]
                rec["sel_ids"], rec["sel_eids"] = rec["ids"], rec["eids"]
                rec["sel_dts"], rec["sel_mask"] = rec["dts"], rec["mask"]
                if "edge_rows" in rec:
                    segs.append((rec["eids"], rec["mask"], rec["B"] * self.budget, rec["edge_rows"]))
                self._node_rows(rec, qv, st)
                rec["queries"] = (qv, qt)
                outs[b].append(rec)
                if rec["layer"] > 1:
                    qs[b] = (rec["next_v"], rec["next_t"])
        if segs:
            arr = (_lib.tg_gather_seg * len(segs))(*[_lib.tg_gather_seg(ptr(e), ptr(mk), n, ptr(o))
                                                     for e, mk, n, o in segs])
            check(_lib.lib.tg_gather_rows_multi(arr, len(segs), estore,
                                                ptr(self.cache.slot_of) if self.cache is not None else None, 0,
                                                row_pitch(g.d_e), st))
        return outs

    def _node_rows(self, rec, qv, st):
        """training.py:223-230 for the selected neighbors (masked -> signed
        zeros) and, for TGAT layer 1, the unmasked target rows."""
        g = self.graph
        if "node_rows" not in rec:
            return
        nstore = feat_store(g.node_features)
        nr = rec["node_rows"]
        n = rec["sel_ids"].numel()
        check(_lib.lib.tg_lookup_gather(ptr(rec["sel_ids"]), ptr(rec["sel_mask"]), n, nstore, None, 1, ptr(nr),
                                        row_pitch(g.d_v), st))
        if "tgt_rows" in rec:
            check(_lib.lib.tg_lookup_gather(ptr(qv), None, int(qv.shape[0]), nstore, None, 0, ptr(rec["tgt_rows"]),
                                            row_pitch(g.d_v), st))

    def join(self, stream=None):
        """Make `stream` (default: current) wait for every in-flight slot."""
        t = _lib.torch()
        cur = stream if stream is not None else t.cuda.current_stream()
        for st in list(self._slot_streams.values()) + list(self._side.values()):
            cur.wait_stream(st)

    def end_epoch(self, group=None):
        """Epoch boundary (training.py:442-443): the cache replacement, after
        every in-flight batch of the epoch.  Under root sharding (a process
        group with more than one rank) the per-edge counters and hit/miss
        stats are first summed across ranks (shard.epoch_allreduce), so every
        rank replaces from the same counts and keeps the resident set -- and
        the reports -- of the 1-GPU run (cache.py:107-118)."""
        if self.cache is None:
            return None
        self.join()
        from .cache import maybe_replace
        from .shard import epoch_allreduce
        epoch_allreduce([self.cache.counters_i32, self.cache.stats], group=group)
        return maybe_replace(self.cache)


class StepGraph:
    """G mini-batch steps of R1 roots captured as ONE CUDA graph.

    A step's host work (argument structs, ctypes calls, stream joins) costs
    more than its device work once the roots are split across ranks (a
    1/8 share of a GDELT batch is ~10 us of HBM time), so the data loader
    replays captured steps instead: ``inputs`` holds, per captured batch j,
    the packed int64 row ``[roots_v (R1) | roots_t as f64 bits (R1) |
    finder seeds (L, layer L first)]``; the finder kernels read their seeds
    from it (``tg_find_args.seed_ptr``), so one copy into ``inputs`` plus one
    ``replay`` runs G whole steps.  The G batches are captured through
    ``generate_batched``: one finder launch per layer covers all of them and
    one K5 launch moves every layer's rows, so their dependent search chains
    overlap inside each grid (graph branches of small per-batch launches ran
    only ~3 at a time).  Outputs
    (``records[j]``, the dicts ``generate`` returns) are valid until the
    next replay.  Cache counting and ``valid`` accumulate exactly as
    ``generate`` does (counts commute).  Non-adaptive configurations only:
    an adaptive layer's K8 draw position is per call.

    ``pack(nodes, times, seeds)`` builds one input row on the host.
    """

    def __init__(self, gen, R1, key, G=1, layer_rows=None, train_mode=True, inputs=None, stream=None):
        t = _lib.torch()
        if gen._adaptive is not None:
            raise ValueError("StepGraph covers non-adaptive layers (an adaptive layer's WOR position is per call)")
        self.gen, self.R1, self.G, self.L = gen, int(R1), int(G), gen.L
        self.width = 2 * self.R1 + self.L
        dev = gen.dev
        # inputs: a caller's [G, width] device block the graph reads in place
        # (``launch()`` then costs one graph launch, no copy); else its own
        self.bound = inputs is not None
        if self.bound and tuple(inputs.shape) != (self.G, self.width):
            raise ValueError(f"inputs must be [{self.G}, {self.width}]")
        self.inputs = inputs if self.bound else t.zeros((self.G, self.width), dtype=t.int64, device=dev)
        self.stream = stream if stream is not None else t.cuda.Stream(device=dev)
        keys = [(key, j) for j in range(self.G)]
        views = []
        for j in range(self.G):
            row = self.inputs[j]
            views.append((row[:self.R1], row[self.R1:2 * self.R1].view(t.float64), row[2 * self.R1:]))
        self._views = views
        # prime lazily initialised state (workspaces, kernel attributes, side
        # streams) outside the capture, without touching the cache counters
        self.stream.wait_stream(t.cuda.current_stream(dev))
        batches = [(views[j][0], views[j][1], views[j][2], keys[j]) for j in range(self.G)]
        with t.cuda.stream(self.stream):
            gen.generate_batched(batches, train_mode=False, layer_rows=layer_rows, stream=self.stream)
        self.stream.synchronize()
        self.graph = t.cuda.CUDAGraph()
        with t.cuda.graph(self.graph, stream=self.stream):
            # the G batches as ONE finder launch per layer + one K5 launch
            # (generate_batched), not G branches of small launches
            recs = gen.generate_batched(batches, train_mode=train_mode, layer_rows=layer_rows,
                                        stream=t.cuda.current_stream(dev))
        self.records = recs
        self._exec = _lib.ctypes.c_void_p(self.graph.raw_cuda_graph_exec())
        self._st = _lib.ctypes.c_void_p(self.stream.cuda_stream)
        check(_lib.lib.tg_graph_upload(self._exec, self._st))  # not on the first replay's clock

    def pack(self, nodes, times, seeds):
        """Host int64 row of one batch: nodes, the bits of times, per-layer seeds."""
        return StepGraph.pack_row(self.R1, self.L, nodes, times, seeds)

    @staticmethod
    def pack_row(R1, L, nodes, times, seeds):
        """``pack`` without a graph: the [2 R1 + L] int64 input row of one batch."""
        import numpy as np
        row = np.empty(2 * R1 + L, dtype=np.int64)
        row[:R1] = np.asarray(nodes, dtype=np.int64)
        row[R1:2 * R1] = np.asarray(times, dtype=np.float64).view(np.int64)
        sd = [int(seeds[l]) if isinstance(seeds, dict) else int(seeds[i]) for i, l in enumerate(range(L, 0, -1))]
        row[2 * R1:] = [x - (1 << 64) if x >= (1 << 63) else x for x in sd]  # u64 bits
        return row

    def replay(self, inputs=None):
        """Run the G captured steps on ``self.stream``; ``inputs`` (device
        int64 [G, width], optional) is copied in first on the same stream.
        The caller's current stream is made to wait for the replay."""
        t = _lib.torch()
        cur = t.cuda.current_stream(self.gen.dev)
        self.stream.wait_stream(cur)
        with t.cuda.stream(self.stream):
            if inputs is not None:
                self.inputs.copy_(inputs, non_blocking=True)
            self.graph.replay()
        cur.wait_stream(self.stream)
        return self.records

    def launch(self, inputs=None):
        """replay() without ordering the caller's stream: batches in flight on
        several StepGraphs overlap; ``wait(stream)`` joins one."""
        t = _lib.torch()
        with t.cuda.stream(self.stream):
            if inputs is not None:
                self.inputs.copy_(inputs, non_blocking=True)
            self.graph.replay()
        return self.records

    def launch_bound(self):
        """Replay a graph built over a caller's inputs block (no input
        copy) on this StepGraph's stream, launching the executable graph
        through the driver (tg_graph_launch): the cheapest host path per G
        steps.  The graph holds no torch RNG state, so bypassing
        CUDAGraph.replay() skips nothing it needs."""
        check(_lib.lib.tg_graph_launch(self._exec, self._st))  # cuGraphLaunch: ~1.5 us vs ~10 for replay()
        return self.records

    def wait(self, stream=None):
        t = _lib.torch()
        (stream if stream is not None else t.cuda.current_stream(self.gen.dev)).wait_stream(self.stream)
