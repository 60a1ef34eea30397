"""Generate golden vectors by running the REAL reference (tgadapt) here.

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

/root/reference is read-only and absent on the GPU box, so its outputs are
frozen into tests/golden/*.npz (small) and the oracle + CUDA path are pinned
against them there.  Numba's cache is redirected so nothing is written into
the reference tree.
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_golden")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

from tgadapt import cache as rcache  # noqa: E402
from tgadapt import finder as rfinder  # noqa: E402
from tgadapt import graph as rgraph  # noqa: E402
from tgadapt import sampler as rsampler  # noqa: E402
from tgadapt import training as rtraining  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _graph_arrays(g):
    return {"offsets": g.tcsr_offsets, "nbr": g.tcsr_neighbors, "adj_ts": g.tcsr_ts, "adj_eid": g.tcsr_eids,
            "src_s": g.src, "dst_s": g.dst, "ts_s": g.ts}


def tcsr_cases(rng):
    cases = {}
    specs = [("sorted", 40, 600, "sorted"), ("unsorted", 60, 900, "unsorted"), ("ties", 30, 700, "ties"),
             ("selfloops", 25, 500, "self"), ("negzero", 12, 80, "negzero"), ("wide", 300, 3000, "unsorted")]
    for name, V, E, kind in specs:
        src = rng.integers(0, V, E)
        dst = rng.integers(0, V, E)
        if kind == "sorted":
            ts = np.sort(rng.random(E) * 100.0)
        elif kind == "unsorted":
            ts = rng.random(E) * 100.0
        elif kind == "ties":
            ts = np.floor(rng.random(E) * E / 8)
        elif kind == "self":
            ts = rng.random(E) * 50.0
            sl = rng.random(E) < 0.1
            dst[sl] = src[sl]
        else:
            ts = np.floor(rng.random(E) * 5)
            ts[rng.random(E) < 0.3] = -0.0
        ef = rng.normal(size=(E, 5)).astype(np.float32)
        g = rgraph.build_graph(src, dst, ts, num_nodes=V + 3, edge_features=ef)
        for k, v in _graph_arrays(g).items():
            cases[f"{name}/{k}"] = v
        cases[f"{name}/in_src"], cases[f"{name}/in_dst"], cases[f"{name}/in_ts"] = src, dst, ts
        cases[f"{name}/in_ef"] = ef
        cases[f"{name}/ef_s"] = g.edge_features
        cases[f"{name}/V"] = np.array(V + 3)
    np.savez_compressed(os.path.join(OUT, "tcsr.npz"), **cases)


def finder_cases(rng):
    cases = {}
    # graph with heavy hubs so that windows span the recent, rejection and
    # complement branches for every m
    V, E = 40, 6000
    src = np.minimum(rng.zipf(1.5, E) - 1, V - 1)
    dst = rng.integers(0, V, E)
    ts = np.floor(rng.random(E) * 3000.0) / 4.0  # ties
    g = rgraph.build_graph(src, dst, ts, num_nodes=V)
    for k, v in _graph_arrays(g).items():
        cases[f"g/{k}"] = v
    cases["g/in_src"], cases["g/in_dst"], cases["g/in_ts"] = src, dst, ts
    B = 3000
    qv = rng.integers(0, V, B)
    qt = rng.random(B) * 800.0
    qt[:50] = ts[rng.integers(0, E, 50)]  # exact-tie query times
    cases["qv"], cases["qt"] = qv, qt
    for m in (1, 3, 10, 25, 60):
        for policy in ("recent", "uniform"):
            for seed in (0, 12345678901234567):
                idx, cnt = rfinder.batch_find_arrays(g, qv, qt, m, policy=policy, seed=seed)
                cases[f"{policy}/m{m}/s{seed}/idx"] = idx
                cases[f"{policy}/m{m}/s{seed}/cnt"] = cnt
    # pivots
    cases["pivot"] = np.array([rfinder.pivot(g, int(v), float(t)) for v, t in zip(qv[:300], qt[:300])])
    np.savez_compressed(os.path.join(OUT, "finder.npz"), **cases)


def cache_cases(rng):
    cases = {}
    for ci, (E, k, eps, epochs) in enumerate([(50, 5, None, 6), (200, 0.2, None, 5), (30, 4, 2, 8), (10, 0, None, 2),
                                              (100, 10, 0.5, 5)]):
        st = rcache.make_cache(E, k, epsilon=eps)
        cases[f"c{ci}/k"], cases[f"c{ci}/eps"] = np.array(st.k), np.array(st.epsilon)
        for ep in range(epochs):
            n = int(rng.integers(0, 400))
            eids = np.minimum(rng.zipf(1.3, n) - 1, E - 1) if ep % 2 else rng.integers(0, E, n)
            cases[f"c{ci}/e{ep}/eids"] = eids
            _, hits = rcache.lookup(st, eids)
            cases[f"c{ci}/e{ep}/hits"] = hits
            cases[f"c{ci}/e{ep}/counters"] = st.counters.copy()
            cases[f"c{ci}/e{ep}/hm"] = np.array([st.epoch_stats[-1].hits, st.epoch_stats[-1].misses])
            cases[f"c{ci}/e{ep}/replaced"] = np.array(rcache.maybe_replace(st))
            cases[f"c{ci}/e{ep}/resident"] = st.resident.copy()
        cases[f"c{ci}/epochs"] = np.array(epochs)
    counts = np.stack([np.bincount(np.minimum(rng.zipf(1.2, 500) - 1, 79), minlength=80) for _ in range(4)])
    cases["oracle/counts"] = counts
    for k in (0, 1, 7, 30, 80):
        r = rcache.oracle_cache(counts, k)
        cases[f"oracle/k{k}"] = np.array([np.nan if x is None else x for x in r])
    np.savez_compressed(os.path.join(OUT, "cache.npz"), **cases)


def wor_cases(rng):
    cases = {}
    for ci, (B, m, n) in enumerate([(400, 25, 10), (300, 10, 10), (200, 7, 3), (150, 60, 20), (100, 130, 12)]):
        mask = rng.random((B, m)) < 0.8
        mask[: B // 10] = False                  # rows with no valid slot
        mask[B // 10: B // 5, :] = False
        mask[B // 10: B // 5, 0] = True          # single valid slot
        logits = rng.normal(size=(B, m)) * 3.0
        from tgadapt import autodiff as ad
        q = ad.softmax_masked(ad.Tensor(logits), mask)
        lq = ad.log_softmax_masked(ad.Tensor(logits), mask)
        pol = rsampler.PolicyOutput(q=q, log_q=lq, mask=mask)
        seed = int(rng.integers(0, 2**31))
        rsampler.sample_without_replacement(pol, n, np.random.default_rng(seed))
        cases[f"w{ci}/q"], cases[f"w{ci}/log_q"], cases[f"w{ci}/mask"] = q.data, lq.data, mask
        cases[f"w{ci}/seed"], cases[f"w{ci}/n"] = np.array(seed), np.array(n)
        cases[f"w{ci}/selected"], cases[f"w{ci}/selected_mask"] = pol.selected, pol.selected_mask
        cases[f"w{ci}/selected_log_q"] = pol.selected_log_q.data
    np.savez_compressed(os.path.join(OUT, "wor.npz"), **cases)


def _trainer_minibatch(trainer, nodes, times, it_key, train_mode=True):
    """The mini-batch half of Trainer._forward (training.py:294-345) with
    the aggregator compute left out; same calls, same order."""
    L = trainer.L
    act = {L: (np.asarray(nodes, dtype=np.int64), np.asarray(times, dtype=np.float64))}
    recs = {}
    for l in range(L, 0, -1):
        tn, tt = act[l]
        rec = trainer._layer_neighborhoods(tn, tt, l, train_mode, it_key)
        recs[l] = rec
        if l > 1:
            w = rec["sel_ids"].shape[1]
            act[l - 1] = (np.concatenate([tn, rec["sel_ids"].ravel()]),
                          np.concatenate([tt, np.repeat(tt, w) - rec["sel_dts"].ravel()]))
    out = {}
    if trainer.cfg.aggregator == "graphmixer":
        r = recs[1]
        out[1] = {"edge_rows": trainer._edge_feature_rows(r["sel_eids"], r["sel_mask"], train_mode),
                  "node_rows": trainer._node_feature_rows(r["sel_ids"], r["sel_mask"])}
    else:
        for l in range(1, L + 1):
            r = recs[l]
            out[l] = {"edge_rows": trainer._edge_feature_rows(r["sel_eids"], r["sel_mask"], train_mode)}
            if l == 1:
                out[l]["node_rows"] = trainer._node_feature_rows(r["sel_ids"], r["sel_mask"])
                out[l]["tgt_rows"] = trainer._node_feature_rows(act[1][0])
    return recs, out, act


def pipeline_cases(rng):
    """Reference Trainer mini-batches on shape-generator graphs (the same
    generator the device path uses), non-adaptive configs A/B-like."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from oracle import shapes as oshapes
    from paper_2402_05396_b200.shapes import SHAPES  # noqa: F401  (spec table only)
    cases = {}
    runs = [("A", dict(aggregator="graphmixer", finder_policy="recent", adaptive_neighbor=False, n=10),
             oshapes_spec("A", 0.02), 3, 0),
            ("B", dict(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=False, n=10),
             oshapes_spec("B", 0.005), 7, 1),
            ("E", dict(aggregator="tgat", finder_policy="recent", adaptive_neighbor=False, n=10),
             oshapes_spec("E", 0.00002), 11, 0),
            ("Bv", dict(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=False, n=6, m=6),
             oshapes_spec("D", 0.002), 5, 2)]
    for tag, kw, spec, gseed, tseed in runs:
        og = oshapes.make_graph(spec, seed=gseed)
        g = rgraph.build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                               edge_features=og.edge_features)
        split = rgraph.chronological_split(g)
        cfg = rtraining.RunConfig(batch_size=64, epochs=1, cache_fraction=0.2, **kw)
        tr = rtraining.Trainer(g, split, cfg, tseed)
        cases[f"{tag}/meta"] = np.array([spec.V, spec.E, spec.d_e, spec.d_v, gseed, tseed, tr.iters_per_epoch])
        its = sorted(set([0, 1, tr.iters_per_epoch // 2, tr.iters_per_epoch - 1]))
        cases[f"{tag}/its"] = np.array(its)
        for ep in range(2):
            for it in its:
                eids = tr.train_eids[(it % tr.iters_per_epoch) * cfg.batch_size:][:cfg.batch_size]
                b = eids.size
                nrng = rtraining.substream(tseed, rtraining._S_NEG, it)
                negs = tr.dst_pool[nrng.integers(0, tr.dst_pool.size, size=b)]
                nodes = np.concatenate([g.src[eids], g.dst[eids], negs])
                times = np.concatenate([g.ts[eids]] * 3)
                recs, fs, act = _trainer_minibatch(tr, nodes, times, it)
                p = f"{tag}/ep{ep}/it{it}"
                cases[p + "/nodes"], cases[p + "/times"] = nodes, times
                for l, r in recs.items():
                    for k in ("sel_ids", "sel_dts", "sel_eids", "sel_mask"):
                        cases[f"{p}/l{l}/{k}"] = r[k]
                    for k, v in fs.get(l, {}).items():
                        if v is not None:
                            # feature buffers are large: keep a digest of the exact f64
                            # bytes plus the first rows verbatim
                            cases[f"{p}/l{l}/{k}_sha"] = np.frombuffer(
                                hashlib.sha256(np.ascontiguousarray(v).tobytes()).digest(), dtype=np.uint8)
                            cases[f"{p}/l{l}/{k}_head"] = np.ascontiguousarray(v).reshape(-1, v.shape[-1])[:16]
                if tr.cache is not None:
                    cases[p + "/counters"] = tr.cache.counters.copy()
            if tr.cache is not None:
                cases[f"{tag}/ep{ep}/hm"] = np.array([tr.cache.epoch_stats[-1].hits, tr.cache.epoch_stats[-1].misses])
                cases[f"{tag}/ep{ep}/replaced"] = np.array(rcache.maybe_replace(tr.cache))
                cases[f"{tag}/ep{ep}/resident"] = tr.cache.resident.copy()
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **cases)


def scoring_cases(rng):
    """Reference encoders + mixer + decoders + masked softmax (the forward
    half of the policy, training.py:269-276) on random candidate blocks,
    with parameters from a real ParamStore."""
    from tgadapt import autodiff as ad
    from tgadapt import encoders as renc
    from tgadapt.params import ParamStore
    cases = {}
    runs = [("s0", 0, 12, 8, 6, "linear", 40), ("s1", 5, 7, 8, 6, "gatv2", 40), ("s2", 5, 0, 8, 5, "gat", 30),
            ("s3", 4, 9, 8, 6, "trans", 30), ("s4", 0, 172, 100, 25, "linear", 24),
            ("s5", 100, 172, 100, 25, "gatv2", 12), ("s6", 0, 266, 100, 25, "trans", 8),
            ("s7", 100, 0, 100, 25, "gat", 8)]
    for tag, d_v, d_e, enc, m, dec, B in runs:
        store_seed = int(rng.integers(0, 2**31))
        span = float(rng.choice([1.0, 1e6]))
        if span > 2.0:
            beta = (enc - 1) / np.log10(span)
            ecfg = renc.EncoderConfig(d_time=enc, d_freq=enc, d_feat=enc, m=m, alpha=10.0, beta=max(beta, 1e-3))
        else:
            ecfg = renc.EncoderConfig.balanced(enc, m)
        scfg = rsampler.SamplerConfig(decoder=dec, n=min(3, m), m=m)
        store = ParamStore(store_seed, dtype=np.float64)
        renc.init_encoder_params(store, ecfg, d_v, d_e)
        d_enc = renc.encoded_width(ecfg, d_v, d_e)
        rsampler.init_sampler_params(store, scfg, d_enc, renc.target_width(ecfg, d_v))
        ids = rng.integers(0, 7, (B, m))
        mask = rng.random((B, m)) < 0.8
        mask[0] = False
        mask[1] = True
        dts = rng.random((B, m)) * span
        dts[2] = 0.0
        node_rows = None if not d_v else (rng.normal(size=(B, m, d_v)).astype(np.float32).astype(np.float64)
                                          * mask[..., None])
        edge_rows = None if not d_e else (rng.normal(size=(B, m, d_e)).astype(np.float32).astype(np.float64)
                                          * mask[..., None])
        tgt = None if not d_v else rng.normal(size=(B, d_v)).astype(np.float32).astype(np.float64)
        z_raw = renc.encode_neighborhood_batch(ids, dts, mask, node_rows, edge_rows, ecfg, store)
        z_mixed = rsampler.mixer_transform(z_raw, mask, store)
        z_t = renc.encode_target_batch(np.arange(B), tgt, ecfg, store)
        pol = rsampler.decode_policy(z_raw, z_mixed, z_t, mask, scfg, ecfg, store, d_v, d_e)
        p = f"{tag}/"
        cases[p + "meta"] = np.array([d_v, d_e, enc, m, B, store_seed])
        cases[p + "decoder"] = np.array(dec)
        cases[p + "ab"] = np.array([ecfg.alpha, ecfg.beta, span])
        cases[p + "ids"], cases[p + "mask"], cases[p + "dts"] = ids, mask, dts
        if d_v:
            cases[p + "node_rows"], cases[p + "tgt_rows"] = node_rows, tgt
        if d_e:
            cases[p + "edge_rows"] = edge_rows
        cases[p + "q"], cases[p + "log_q"] = pol.q.data, pol.log_q.data
        if enc <= 8:
            cases[p + "z_raw"], cases[p + "z_mixed"], cases[p + "z_target"] = z_raw.data, z_mixed.data, z_t.data
        h = hashlib.sha256()
        for name in sorted(store.names()):
            h.update(name.encode())
            h.update(np.ascontiguousarray(store[name].data).tobytes())
        cases[p + "params_sha"] = np.frombuffer(h.digest(), dtype=np.uint8)
        if enc <= 8:
            for name in store.names():
                cases[p + "param/" + name] = store[name].data
    np.savez_compressed(os.path.join(OUT, "scoring.npz"), **cases)


def adaptive_cases(rng):
    """Reference Trainer mini-batches with the adaptive sampler on
    (training.py:255-292): candidates, q/log q, selections, cache state."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from oracle import shapes as oshapes
    cases = {}
    runs = [("C", dict(aggregator="graphmixer", finder_policy="recent", decoder="linear"), oshapes_spec("C", 0.0004),
             13, 0, 48),
            ("D", dict(aggregator="tgat", finder_policy="uniform", decoder="gatv2"), oshapes_spec("D", 0.002), 5, 1,
             16),
            ("Dt", dict(aggregator="tgat", finder_policy="recent", decoder="trans"), oshapes_spec("D", 0.001), 6, 2,
             12),
            ("Cg", dict(aggregator="graphmixer", finder_policy="uniform", decoder="gat", m=12, n=5),
             oshapes_spec("D", 0.001), 8, 3, 24)]
    for tag, kw, spec, gseed, tseed, batch in runs:
        og = oshapes.make_graph(spec, seed=gseed)
        g = rgraph.build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                               edge_features=og.edge_features)
        split = rgraph.chronological_split(g)
        cfg = rtraining.RunConfig(batch_size=batch, epochs=1, cache_fraction=0.2, adaptive_neighbor=True,
                                  adaptive_minibatch=False, **kw)
        tr = rtraining.Trainer(g, split, cfg, tseed)
        cases[f"{tag}/meta"] = np.array([spec.V, spec.E, spec.d_e, spec.d_v, gseed, tseed, tr.iters_per_epoch,
                                         batch, cfg.m, cfg.n])
        cases[f"{tag}/ab"] = np.array([tr.ecfg.alpha, tr.ecfg.beta, tr.time_span])
        h = hashlib.sha256()
        for name in sorted(tr.sampler_store.names()):
            h.update(name.encode())
            h.update(np.ascontiguousarray(tr.sampler_store[name].data).tobytes())
        cases[f"{tag}/params_sha"] = np.frombuffer(h.digest(), dtype=np.uint8)
        its = sorted(set([0, tr.iters_per_epoch // 2, tr.iters_per_epoch - 1]))
        cases[f"{tag}/its"] = np.array(its)
        for it in its:
            eids = tr.train_eids[(it % tr.iters_per_epoch) * cfg.batch_size:][:cfg.batch_size]
            b = eids.size
            nrng = rtraining.substream(tseed, rtraining._S_NEG, it)
            negs = tr.dst_pool[nrng.integers(0, tr.dst_pool.size, size=b)]
            nodes = np.concatenate([g.src[eids], g.dst[eids], negs])
            times = np.concatenate([g.ts[eids]] * 3)
            recs, fs, act = _trainer_minibatch(tr, nodes, times, it)
            p = f"{tag}/it{it}"
            cases[p + "/nodes"], cases[p + "/times"] = nodes, times
            for l, r in recs.items():
                for k in ("sel_ids", "sel_dts", "sel_eids", "sel_mask"):
                    cases[f"{p}/l{l}/{k}"] = r[k]
                pol = r["policy"]
                cases[f"{p}/l{l}/q"], cases[f"{p}/l{l}/log_q"] = pol.q.data, pol.log_q.data
                cases[f"{p}/l{l}/cand_mask"] = pol.mask
                cases[f"{p}/l{l}/selected"] = pol.selected
                cases[f"{p}/l{l}/selected_log_q"] = pol.selected_log_q.data
                for k, v in fs.get(l, {}).items():
                    if v is not None:
                        cases[f"{p}/l{l}/{k}_sha"] = np.frombuffer(
                            hashlib.sha256(np.ascontiguousarray(v).tobytes()).digest(), dtype=np.uint8)
            if tr.cache is not None:
                cases[p + "/counters"] = tr.cache.counters.copy()
                cases[p + "/hm"] = np.array([tr.cache.epoch_stats[-1].hits, tr.cache.epoch_stats[-1].misses])
    np.savez_compressed(os.path.join(OUT, "adaptive.npz"), **cases)


def selector_cases(rng):
    """select_batch / update_scores of the real selector (selector.py:36-61)
    with the Trainer's stream (training.py:364-367: substream(seed, S_BATCH, it))."""
    from tgadapt import selector as rsel
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    from oracle.selector import SELECTOR_CASES, case_scores as selector_scores
    cases = {}
    for ci, (kind, n, b, seed) in enumerate(SELECTOR_CASES):
        skind = "random" if kind == "few" else kind
        scores = rsel.ImportanceScores(selector_scores(skind, n, seed), 0.1, base_eid=1000)
        for it in range(3):
            stream = rtraining.substream(seed, rtraining._S_BATCH, it)
            st = stream.bit_generator.state["state"]
            eids = rsel.select_batch(scores, b, stream)
            p = f"c{ci}/it{it}"
            cases[p + "/eids"] = eids
            cases[p + "/pcg"] = np.array([st["state"] >> 64, st["state"] & (2**64 - 1), st["inc"] >> 64,
                                          st["inc"] & (2**64 - 1)], dtype=np.uint64)
            logits = np.random.default_rng(seed * 7 + it).normal(size=b) * 4
            rsel.update_scores(scores, eids, logits)
            cases[p + "/logits"] = logits
            if n <= 20000:
                cases[p + "/scores_after"] = scores.scores.copy()
            else:
                cases[p + "/scores_after_sha"] = np.frombuffer(
                    hashlib.sha256(scores.scores.tobytes()).digest(), dtype=np.uint8)
        cases[f"c{ci}/meta"] = np.array([n, b, seed, 1000])
        cases[f"c{ci}/kind"] = np.array(skind)
    # the Trainer's own non-adaptive start: init_scores
    cases["init_scores"] = rsel.init_scores(17, gamma=0.25).scores
    np.savez_compressed(os.path.join(OUT, "selector.npz"), **cases)


def matio_cases(rng):
    """FMAT files written by the reference's save_matrix (matio.py:27-36)."""
    from tgadapt import matio as rmatio
    rmatio.save_matrix(os.path.join(OUT, "feat_f32.fmat"), rng.normal(size=(37, 13)).astype(np.float32))
    rmatio.save_matrix(os.path.join(OUT, "feat_f64.fmat"), rng.normal(size=(9, 5)))


def aggregator_cases(rng):
    """GraphMixer aggregator forward (training.py:318-330): build_messages
    (aggregators.py:58-71) -> graphmixer_layer (aggregators.py:140-145:
    mixer_forward + mean over slots) with a real model ParamStore."""
    from tgadapt import aggregators as ragg
    from tgadapt import autodiff as rad
    from tgadapt.params import ParamStore
    cases = {}
    runs = [("g0", 0, 172, 100, 10, 40, 1e6), ("g1", 100, 172, 100, 10, 24, 1e6), ("g2", 0, 266, 100, 10, 16, 1.0),
            ("g3", 12, 0, 20, 7, 30, 1e3), ("g4", 0, 186, 100, 25, 8, 1e6)]
    for tag, d_v, d_e, d_time, n, B, span in runs:
        seed = int(rng.integers(0, 2**31))
        for prec in ("float64", "float32"):
            store = ParamStore(seed, dtype=np.dtype(prec))
            ragg.init_time_encode_params(store, d_time, time_span=span)
            d_msg = d_v + d_e + d_time
            ragg.init_graphmixer_params(store, n, d_msg)
            # non-trivial vectors (a trained store's LN affine terms, biases,
            # time phases); the matrices keep their seeded Glorot init
            rv = np.random.default_rng(seed + 1)
            for name in sorted(store.names()):
                if store[name].data.ndim == 1 and name != "model/time_w":
                    store[name].data[...] = rv.normal(size=store[name].data.shape) * 0.3 + (
                        1.0 if name.endswith("gamma") else 0.0)
            r2 = np.random.default_rng(seed)
            mask = r2.random((B, n)) < 0.75
            mask[0] = False
            mask[1] = True
            dts = r2.random((B, n)) * span
            node_rows = None if not d_v else (r2.normal(size=(B, n, d_v)).astype(np.float32).astype(prec)
                                             * mask[..., None])
            edge_rows = None if not d_e else (r2.normal(size=(B, n, d_e)).astype(np.float32).astype(prec)
                                             * mask[..., None])
            h_prev = rad.Tensor(node_rows if node_rows is not None else np.zeros((B, n, 0), dtype=prec))
            msgs = ragg.build_messages(h_prev, edge_rows, dts, mask, store, d_time)
            h = ragg.graphmixer_layer(msgs, store)
            p = f"{tag}/{prec}/"
            cases[p + "h"] = h.data
            if prec == "float64":
                cases[f"{tag}/meta"] = np.array([d_v, d_e, d_time, n, B, seed])
                cases[f"{tag}/span"] = np.array(span)
                cases[f"{tag}/mask"] = mask
                cases[f"{tag}/dts"] = dts
                if node_rows is not None:
                    cases[f"{tag}/node_rows"] = node_rows.astype(np.float32)
                if edge_rows is not None:
                    cases[f"{tag}/edge_rows"] = edge_rows.astype(np.float32)
                for name in store.names():
                    a = store[name].data
                    if a.ndim == 1:
                        cases[f"{tag}/param/{name}"] = a
                    else:  # Glorot matrices are regenerated from (seed, name); pin them by hash
                        cases[f"{tag}/sha/{name}"] = np.frombuffer(hashlib.sha256(a.tobytes()).digest(),
                                                                   dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "aggregator.npz"), **cases)


def tgat_cases(rng):
    """Two TGAT layers (aggregators.py:74-132 tgat_layer, build_messages
    :58-71; the Trainer's bottom-up order training.py:333-356) on random
    layer buffers with a real model ParamStore."""
    from tgadapt import aggregators as ragg
    from tgadapt import autodiff as rad
    from tgadapt.params import ParamStore
    cases = {}
    runs = [("t0", 0, 186, 100, 100, 10, 12, 1e6), ("t1", 100, 172, 100, 100, 10, 8, 1e6),
            ("t2", 0, 0, 16, 24, 5, 20, 50.0), ("t3", 12, 30, 20, 32, 25, 6, 1e3)]
    for tag, d_v, d_e, d_time, d, n, B, span in runs:
        seed = int(rng.integers(0, 2**31))
        B1 = B * (1 + n)
        r2 = np.random.default_rng(seed)
        mask1 = r2.random((B1, n)) < 0.7
        mask1[0] = False
        mask2 = r2.random((B, n)) < 0.8
        mask2[1] = False
        dts1 = r2.random((B1, n)) * span
        dts2 = r2.random((B, n)) * span
        nbr_rows = (r2.normal(size=(B1, n, d_v)).astype(np.float32) * mask1[..., None]) if d_v else None
        tgt_rows = r2.normal(size=(B1, d_v)).astype(np.float32) if d_v else None
        e1 = (r2.normal(size=(B1, n, d_e)).astype(np.float32) * mask1[..., None]) if d_e else None
        e2 = (r2.normal(size=(B, n, d_e)).astype(np.float32) * mask2[..., None]) if d_e else None
        cases[f"{tag}/meta"] = np.array([d_v, d_e, d_time, d, n, B, seed])
        cases[f"{tag}/span"] = np.array(span)
        for k, v in (("mask1", mask1), ("mask2", mask2), ("dts1", dts1), ("dts2", dts2), ("nbr_rows", nbr_rows),
                     ("tgt_rows", tgt_rows), ("e1", e1), ("e2", e2)):
            if v is not None:
                cases[f"{tag}/{k}"] = v
        for prec in ("float64", "float32"):
            store = ParamStore(seed, dtype=np.dtype(prec))
            ragg.init_time_encode_params(store, d_time, time_span=span)
            ragg.init_tgat_params(store, 1, d_v, d_v + d_e + d_time, d)
            ragg.init_tgat_params(store, 2, d, d + d_e + d_time, d)
            rv = np.random.default_rng(seed + 1)
            for name in sorted(store.names()):
                if store[name].data.ndim == 1 and name != "model/time_w":
                    store[name].data[...] = rv.normal(size=store[name].data.shape) * 0.3
            cast = lambda a: None if a is None else a.astype(prec)  # noqa: E731
            h_nbr = rad.Tensor(cast(nbr_rows) if d_v else np.zeros((B1, n, 0), dtype=prec))
            h_tgt = rad.Tensor(cast(tgt_rows) if d_v else np.zeros((B1, 0), dtype=prec))
            m1 = ragg.build_messages(h_nbr, cast(e1), dts1, mask1, store, d_time)
            h1, tau1, _ = ragg.tgat_layer(h_tgt, m1, mask1, store, 1, d_e)
            h_tgt2 = rad.index(h1, (slice(0, B),))
            h_nbr2 = rad.reshape(rad.index(h1, (slice(B, None),)), (B, n, d))
            m2 = ragg.build_messages(h_nbr2, cast(e2), dts2, mask2, store, d_time)
            h2, tau2, _ = ragg.tgat_layer(h_tgt2, m2, mask2, store, 2, d_e)
            p = f"{tag}/{prec}/"
            cases[p + "h1"] = h1.data
            cases[p + "tau1"] = tau1.data
            cases[p + "h2"] = h2.data
            cases[p + "tau2"] = tau2.data
            if prec == "float64":
                for name in store.names():
                    a = store[name].data
                    if a.ndim == 1:
                        cases[f"{tag}/param/{name}"] = a
                    else:
                        cases[f"{tag}/sha/{name}"] = np.frombuffer(hashlib.sha256(a.tobytes()).digest(),
                                                                   dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "tgat.npz"), **cases)


INGEST_FILES = {
    "crlf.csv": "0,1,0.5,1.0,2.0\r\n1,2,1.5,-0.0,3e-5\r\n# comment\r\n\r\n2,0,2.0,1_000.25,inf\r\n",
    "cr.csv": "  0 , 1 , 1e3 , 7\r1,2,+2.5e-3,-nan\r3,4,00012.5,1E+2",
    "plain.csv": "5,6,0.1\n6,7,0.2\n#x,y,z\n7,8,1.7976931348623157e308\n8,9,4.9e-324\n",
    "wide.csv": "".join(f"{i % 13},{(i * 7) % 13},{i * 0.37!r},{','.join(repr(float(np.float32(np.sin(i * j))))
                                                          for j in range(40))}\n" for i in range(300)),
    "err_few.csv": "0,1,0.5\n1,2\n",
    "err_int.csv": "0,1,0.5\n1.5,2,3.0\n",
    "err_float.csv": "0,1,0.5,1.0\n1,2,3.0,abc\n",
    "err_nonfinite.csv": "0,1,0.5\n1,2,nan\n",
    "err_width.csv": "0,1,0.5,1.0,2.0\n1,2,3.0,1.0\n",
}


def ingest_cases(rng):
    """Event files read by the reference's ingest_events / load_manifest
    (graph.py:159-222), including a dataset written by save_dataset."""
    from tgadapt import graph as rg
    d = os.path.join(OUT, "ingest")
    os.makedirs(d, exist_ok=True)
    cases = {}
    for name, text in INGEST_FILES.items():
        with open(os.path.join(d, name), "w", newline="") as fh:
            fh.write(text)
        try:
            g = rg.ingest_events(os.path.join(d, name))
            cases[f"{name}/src"] = g.src
            cases[f"{name}/dst"] = g.dst
            cases[f"{name}/ts"] = g.ts
            if g.edge_features is not None:
                cases[f"{name}/ef"] = g.edge_features
            cases[f"{name}/offsets"] = g.tcsr_offsets
        except rg.DataError as exc:
            cases[f"{name}/error"] = np.array(str(exc).replace(d + "/", ""))
    # a dataset written by the reference itself (repr floats, FMAT node features)
    V, E = 50, 700
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    ts = np.sort(rng.random(E) * 1e6)
    ef = rng.normal(size=(E, 9)).astype(np.float32)
    nf = rng.normal(size=(V, 4)).astype(np.float32)
    g0 = rg.build_graph(src, dst, ts, num_nodes=V, node_features=nf, edge_features=ef)
    mpath = rg.save_dataset(g0, d, name="ds")
    g = rg.load_manifest(mpath)
    for k in ("src", "dst", "ts", "tcsr_offsets", "tcsr_neighbors", "tcsr_eids", "tcsr_ts", "edge_features",
              "node_features"):
        cases[f"ds/{k}"] = getattr(g, k)
    np.savez_compressed(os.path.join(OUT, "ingest.npz"), **cases)


def surrogate_cases(rng):
    """Surrogate-loss head (sampler.py:183-250, training.py:409-436): the
    coefficients, the loss and, through ad.backward, d loss / d logits."""
    from tgadapt import autodiff as ad
    cases = {}
    shapes = [(150, 25, 10, 40, 60, 20), (120, 10, 10, 16, 33, 7), (40, 60, 20, 64, 96, 50), (50, 7, 3, 5, 9, 3)]
    for ci, (B, m, n, d, dm, ht) in enumerate(shapes):
        for dt in (np.float64, np.float32):
            tag = f"s{ci}_{'f64' if dt == np.float64 else 'f32'}"
            mask = rng.random((B, m)) < 0.8
            mask[: B // 10] = False
            mask[B // 10: B // 5, :] = False
            mask[B // 10: B // 5, 0] = True
            logits_np = (rng.normal(size=(B, m)) * 2.0).astype(dt)
            contrib = rng.random(B) < 0.9
            dL = rng.normal(size=(B, d)).astype(dt)
            out = {"mask": mask, "contrib": contrib, "dL_dh": dL}
            for agg in ("tgat", "graphmixer"):
                logits = ad.Tensor(logits_np.copy(), requires_grad=True)
                q = ad.softmax_masked(logits, mask)
                lq = ad.log_softmax_masked(logits, mask)
                pol = rsampler.PolicyOutput(q=q, log_q=lq, mask=mask)
                seed = int(rng.integers(0, 2**31))
                rsampler.sample_without_replacement(pol, n, np.random.default_rng(seed))
                sel, smask = pol.selected, pol.selected_mask
                if agg == "tgat":
                    tau = np.exp(rng.normal(size=(B, n))).astype(dt)
                    V = rng.normal(size=(B, n, d)).astype(dt)
                    c = rsampler.tgat_sample_coefficients(ad.Tensor(dL), ad.Tensor(tau), ad.Tensor(V), smask, contrib)
                    loss = rsampler.sample_loss_tgat(ad.Tensor(dL), ad.Tensor(tau), ad.Tensor(V), pol.selected_log_q,
                                                     sel_mask=smask, contrib_mask=contrib)
                    out.update({"tau": tau, "V": V})
                    # the reference formula evaluated in f64 on the same inputs: its
                    # float32 run loses up to a few % to cancellation between the
                    # two quotient-rule terms, so f32 parity is judged against this
                    out["tgat/c64"] = rsampler.tgat_sample_coefficients(
                        ad.Tensor(dL.astype(np.float64)), ad.Tensor(tau.astype(np.float64)),
                        ad.Tensor(V.astype(np.float64)), smask, contrib)
                else:
                    msgs = rng.normal(size=(B, n, dm)).astype(dt)
                    Wc1 = (rng.normal(size=(dm, d)) / np.sqrt(dm)).astype(dt)
                    Wt1 = (rng.normal(size=(n, ht)) / np.sqrt(n)).astype(dt)
                    Wt2 = (rng.normal(size=(ht, n)) / np.sqrt(ht)).astype(dt)
                    mu = msgs @ Wc1                                  # training.py:425-428
                    w_row = 1.0 + (Wt1 @ Wt2).sum(axis=1)
                    w_prime = np.broadcast_to(w_row[None, :, None], mu.shape)
                    c = rsampler.graphmixer_sample_coefficients(dL, w_prime, mu, smask, contrib)
                    loss = rsampler.sample_loss_graphmixer(dL, w_prime, mu, pol.selected_log_q,
                                                           sel_mask=smask, contrib_mask=contrib)
                    out.update({"msgs": msgs, "Wc1": Wc1, "Wt1": Wt1, "Wt2": Wt2, "w_row": w_row})
                ad.backward(loss)
                out.update({f"{agg}/q": q.data, f"{agg}/log_q": lq.data, f"{agg}/selected": sel,
                            f"{agg}/sel_mask": smask, f"{agg}/c": c, f"{agg}/loss": np.array(loss.data),
                            f"{agg}/dlogits": logits.grad})
            for k, v in out.items():
                cases[f"{tag}/{k}"] = v
    np.savez_compressed(os.path.join(OUT, "surrogate.npz"), **cases)


def sampler_grad_cases(rng):
    """The scoring network's backward: the reference
    forward (encoders -> mixer -> decoder -> masked (log-)softmax, as
    training.py:269-276 runs it), WOR picks, a surrogate loss
    sum(c * selected_log_q) (sample_loss_*, sampler.py:216-250) and
    ad.backward -> every sampler parameter's .grad.  d loss / d logits is
    restated here from the reference's q (index + log_softmax_masked vjp,
    autodiff.py:257-271, 447-464) as the input of the device backward."""
    from tgadapt import autodiff as ad
    from tgadapt import encoders as renc
    from tgadapt.params import ParamStore
    cases = {}
    runs = [("g0", 0, 12, 8, 6, "linear", 20), ("g1", 5, 7, 8, 6, "gatv2", 20), ("g2", 5, 0, 8, 5, "gat", 16),
            ("g3", 4, 9, 8, 6, "trans", 16), ("g4", 6, 0, 12, 10, "linear", 12), ("g5", 0, 5, 8, 7, "gat", 14),
            ("g6", 3, 4, 6, 9, "gatv2", 10), ("g7", 0, 172, 100, 25, "linear", 6)]
    for tag, d_v, d_e, enc, m, dec, B in runs:
        store_seed = int(rng.integers(0, 2**31))
        span = 1e6
        beta = (enc - 1) / np.log10(span)
        ecfg = renc.EncoderConfig(d_time=enc, d_freq=enc, d_feat=enc, m=m, alpha=10.0, beta=beta)
        n = min(4, m)
        scfg = rsampler.SamplerConfig(decoder=dec, n=n, m=m)
        store = ParamStore(store_seed, dtype=np.float64)
        renc.init_encoder_params(store, ecfg, d_v, d_e)
        d_enc = renc.encoded_width(ecfg, d_v, d_e)
        rsampler.init_sampler_params(store, scfg, d_enc, renc.target_width(ecfg, d_v))
        # perturb the zero / one initialised affine terms so every vjp is exercised
        for name in store.names():
            if name.endswith(("bc1", "bc2", "bt1", "bt2", "beta")):
                store[name].data[...] = rng.normal(size=store[name].data.shape) * 0.1
            elif name.endswith("gamma"):
                store[name].data[...] = 1.0 + rng.normal(size=store[name].data.shape) * 0.1
        ids = rng.integers(0, 5, (B, m))
        mask = rng.random((B, m)) < 0.8
        mask[0] = False
        mask[1] = True
        dts = rng.random((B, m)) * span
        node_rows = None if not d_v else (rng.normal(size=(B, m, d_v)).astype(np.float32).astype(np.float64)
                                          * mask[..., None])
        edge_rows = None if not d_e else (rng.normal(size=(B, m, d_e)).astype(np.float32).astype(np.float64)
                                          * mask[..., None])
        tgt = None if not d_v else rng.normal(size=(B, d_v)).astype(np.float32).astype(np.float64)
        store.zero_grad()
        z_raw = renc.encode_neighborhood_batch(ids, dts, mask, node_rows, edge_rows, ecfg, store)
        z_mixed = rsampler.mixer_transform(z_raw, mask, store)
        z_t = renc.encode_target_batch(np.arange(B), tgt, ecfg, store)
        pol = rsampler.decode_policy(z_raw, z_mixed, z_t, mask, scfg, ecfg, store, d_v, d_e)
        rsampler.sample_without_replacement(pol, n, np.random.default_rng(int(rng.integers(0, 2**31))))
        c = rng.normal(size=(B, n)) * pol.selected_mask
        loss = ad.sum_all(ad.mul(pol.selected_log_q, ad.Tensor(c)))
        ad.backward(loss)
        # d loss / d logits: scatter c into the picks, then the log-softmax vjp
        q = pol.q.data
        dlq = np.zeros((B, m))
        rows = np.repeat(np.arange(B)[:, None], n, axis=1)
        np.add.at(dlq, (rows, np.maximum(pol.selected, 0)), c * pol.selected_mask)
        gm = np.where(mask, dlq, 0.0)
        dlogits = gm - q * gm.sum(axis=-1, keepdims=True)
        p = f"{tag}/"
        cases[p + "meta"] = np.array([d_v, d_e, enc, m, B, store_seed, n])
        cases[p + "decoder"] = np.array(dec)
        cases[p + "ab"] = np.array([ecfg.alpha, ecfg.beta, span])
        cases[p + "ids"], cases[p + "mask"], cases[p + "dts"] = ids, mask, dts
        if d_v:
            cases[p + "node_rows"], cases[p + "tgt_rows"] = node_rows, tgt
        if d_e:
            cases[p + "edge_rows"] = edge_rows
        cases[p + "q"], cases[p + "dlogits"] = q, dlogits
        cases[p + "selected"], cases[p + "sel_mask"], cases[p + "c"] = pol.selected, pol.selected_mask, c
        for name in store.names():
            if name.endswith(("bc1", "bc2", "bt1", "bt2", "beta", "gamma")):  # the rest: sampler_params(store_seed)
                cases[p + "param/" + name] = store[name].data
            g = store[name].grad
            cases[p + "grad/" + name] = np.zeros_like(store[name].data) if g is None else g
    np.savez_compressed(os.path.join(OUT, "sampler_grad.npz"), **cases)


def adam_cases(rng):
    """ParamStore.adam_step (params.py:80-99): three steps on a small store,
    float64 and float32 (one float32 parameter gets a float64 gradient, one
    step leaves a parameter without gradient)."""
    from tgadapt import params as rparams
    cases = {}
    shapes = {"a": (7, 5), "b": (13,), "c": (3, 4, 2), "d": (300,)}
    for dt, tag in ((np.float64, "f64"), (np.float32, "f32")):
        store = rparams.ParamStore(seed=int(rng.integers(0, 2**31)), dtype=dt)
        for k, shp in shapes.items():
            store.glorot(f"sampler/{k}", shp)
        for k in shapes:
            cases[f"{tag}/init/{k}"] = store[f"sampler/{k}"].data.copy()
        hp = [(1e-3, 0.9, 0.999, 1e-8), (5e-2, 0.8, 0.99, 1e-6), (1e-3, 0.9, 0.999, 1e-8)]
        for step, (lr, b1, b2, eps) in enumerate(hp):
            for k, shp in shapes.items():
                if step == 1 and k == "b":
                    g = None
                else:
                    g = rng.normal(size=shp) * 10.0 ** rng.integers(-6, 2)
                    g = g.astype(np.float64 if (tag == "f32" and k == "c") else dt)
                store[f"sampler/{k}"].grad = g
                cases[f"{tag}/s{step}/g/{k}"] = g if g is not None else np.zeros(0)
            store.adam_step(lr, beta1=b1, beta2=b2, eps=eps)
            cases[f"{tag}/s{step}/hp"] = np.array([lr, b1, b2, eps])
            for k in shapes:
                cases[f"{tag}/s{step}/p/{k}"] = store[f"sampler/{k}"].data.copy()
                cases[f"{tag}/s{step}/m/{k}"] = store._adam_m[f"sampler/{k}"].copy()
                cases[f"{tag}/s{step}/v/{k}"] = store._adam_v[f"sampler/{k}"].copy()
    np.savez_compressed(os.path.join(OUT, "adam.npz"), **cases)


def oshapes_spec(key, factor):
    from paper_2402_05396_b200.shapes import SHAPES
    return SHAPES[key].scaled(factor)


if __name__ == "__main__":
    which = sys.argv[1:] or ["tcsr", "finder", "cache", "wor", "pipeline", "scoring", "adaptive", "selector", "matio", "aggregator", "tgat", "ingest", "surrogate", "adam", "sampler_grad"]
    rng = np.random.default_rng(20240207)
    # one independent stream per case family (fixed order), so regenerating
    # one family does not disturb the others
    streams = {w: rng.integers(0, 2**31) for w in ["tcsr", "finder", "cache", "wor", "pipeline", "scoring",
                                                   "adaptive", "selector", "matio", "aggregator", "tgat", "ingest",
                                                   "surrogate", "adam", "sampler_grad"]}
    for w in which:
        globals()[f"{w}_cases"](np.random.default_rng(streams[w]))
        print("wrote", w)
