"""Parity of the sm_100a kernels (through the C-ABI) against the golden
vectors of the real reference and the CPU oracle.  Bit-exact for every
integer / index / copy result; run with ``pytest -m gpu`` on a B200."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

TCSR_CASES = ["sorted", "unsorted", "ties", "selfloops", "negzero", "wide"]


def _np(x):
    return x.detach().cpu().numpy()


def _sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8)


def _dev_graph_from_golden(z, prefix):
    import torch
    from paper_2402_05396_b200.graph import from_device_tcsr
    c = lambda k, dt: torch.as_tensor(z[f"{prefix}/{k}"]).to("cuda", dt)  # noqa: E731
    return from_device_tcsr(z[f"{prefix}/offsets"].shape[0] - 1, c("src_s", torch.int64), c("dst_s", torch.int64),
                            c("ts_s", torch.float64), c("offsets", torch.int64), c("nbr", torch.int32),
                            c("adj_ts", torch.float64), c("adj_eid", torch.int32))


# ---------------------------------------------------------------- K1 T-CSR
@pytest.mark.parametrize("case", TCSR_CASES)
def test_device_tcsr_bit_exact(case):
    from paper_2402_05396_b200 import build_graph
    z = load_golden("tcsr")
    g = build_graph(z[f"{case}/in_src"], z[f"{case}/in_dst"], z[f"{case}/in_ts"], num_nodes=int(z[f"{case}/V"]),
                    edge_features=z[f"{case}/in_ef"])
    np.testing.assert_array_equal(_np(g.tcsr_offsets), z[f"{case}/offsets"])
    np.testing.assert_array_equal(_np(g.tcsr_neighbors), z[f"{case}/nbr"])
    np.testing.assert_array_equal(_np(g.tcsr_eids), z[f"{case}/adj_eid"])
    np.testing.assert_array_equal(_np(g.src), z[f"{case}/src_s"])
    np.testing.assert_array_equal(_np(g.dst), z[f"{case}/dst_s"])
    assert _np(g.tcsr_ts).tobytes() == z[f"{case}/adj_ts"].tobytes()
    assert _np(g.ts).tobytes() == z[f"{case}/ts_s"].tobytes()
    assert _np(g.edge_features).tobytes() == z[f"{case}/ef_s"].tobytes()


def test_device_tcsr_validation():
    from paper_2402_05396_b200 import DataError, build_graph
    with pytest.raises(DataError, match="length mismatch"):
        build_graph([0, 1], [1], [0.0, 1.0])
    with pytest.raises(DataError, match="non-finite"):
        build_graph([0, 1], [1, 0], [1.0, np.inf])
    with pytest.raises(DataError, match="negative timestamp"):
        build_graph([0], [1], [-1.0])
    with pytest.raises(DataError, match="negative node"):
        build_graph([0], [-1], [1.0])
    with pytest.raises(DataError, match="num_nodes"):
        build_graph([0], [5], [1.0], num_nodes=3)
    with pytest.raises(DataError, match="edge feature"):
        build_graph([0], [1], [1.0], edge_features=np.zeros((2, 3), np.float32))
    g = build_graph([], [], [], num_nodes=4)
    assert g.num_events == 0 and _np(g.tcsr_offsets).tolist() == [0] * 5


def test_device_tcsr_large_matches_oracle():
    """4M events, tie-heavy unsorted ts (exercises both radix sorts)."""
    from oracle import shapes as oshapes
    from oracle import tcsr as otcsr
    from paper_2402_05396_b200 import build_graph
    src, dst, ts = oshapes.synth_events(5000, 4_000_000, 9, ts_mode=1)
    og = otcsr.build_graph(src, dst, ts, num_nodes=5000)
    g = build_graph(src, dst, ts, num_nodes=5000)
    np.testing.assert_array_equal(_np(g.tcsr_offsets), og.tcsr_offsets)
    np.testing.assert_array_equal(_np(g.nbr32), og.tcsr_neighbors)
    np.testing.assert_array_equal(_np(g.eid32), og.tcsr_eids)
    assert _np(g.tcsr_ts).tobytes() == og.tcsr_ts.tobytes()


def test_device_synth_matches_host_twin():
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import shapes
    for mode in (0, 1, 2):
        s, d, t = shapes.synth_events_device(777, 50_000, 21, ts_mode=mode)
        hs, hd, ht = oshapes.synth_events(777, 50_000, 21, ts_mode=mode)
        np.testing.assert_array_equal(_np(s), hs)
        np.testing.assert_array_equal(_np(d), hd)
        assert _np(t).tobytes() == ht.tobytes()
    f = shapes.synth_features_device(3000, 186, 5)
    assert _np(f).tobytes() == oshapes.synth_features(0, 3000, 186, 5).tobytes()
    torch.cuda.synchronize()


# ---------------------------------------------------------------- K2 finder
@pytest.mark.parametrize("policy", ["recent", "uniform"])
@pytest.mark.parametrize("m", [1, 3, 10, 25, 60])
@pytest.mark.parametrize("seed", [0, 12345678901234567])
def test_device_finder_bit_exact(policy, m, seed):
    from paper_2402_05396_b200 import batch_find_arrays
    z = load_golden("finder")
    g = _dev_graph_from_golden(z, "g")
    idx, cnt = batch_find_arrays(g, z["qv"], z["qt"], m, policy=policy, seed=seed)
    np.testing.assert_array_equal(idx, z[f"{policy}/m{m}/s{seed}/idx"])
    np.testing.assert_array_equal(cnt, z[f"{policy}/m{m}/s{seed}/cnt"])


def test_device_pivot_and_sharded_rows():
    import torch
    from paper_2402_05396_b200 import batch_find_arrays, pivot
    z = load_golden("finder")
    g = _dev_graph_from_golden(z, "g")
    assert [pivot(g, int(v), float(t)) for v, t in zip(z["qv"][:100], z["qt"][:100])] == list(z["pivot"][:100])
    # a shard of rows [a, b) keyed by row_base reproduces the full batch
    qv = torch.as_tensor(z["qv"]).cuda()
    qt = torch.as_tensor(z["qt"]).cuda()
    full, _ = batch_find_arrays(g, qv, qt, 10, policy="uniform", seed=77)
    a, b = 1000, 2300
    part, _ = batch_find_arrays(g, qv[a:b], qt[a:b], 10, policy="uniform", seed=77, row_base=a)
    assert torch.equal(full[a:b], part)


def test_device_finder_large_vs_oracle():
    """Hub windows far above 128 entries (multi-round 32-ary pivot search)."""
    from oracle import finder as ofinder
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import batch_find_arrays, build_graph
    src, dst, ts = oshapes.synth_events(300, 2_000_000, 4, ts_mode=0)
    from oracle import tcsr as otcsr
    og = otcsr.build_graph(src, dst, ts, num_nodes=300)
    g = build_graph(src, dst, ts, num_nodes=300)
    rng = np.random.default_rng(0)
    qv = rng.integers(0, 300, 20000)
    qt = rng.random(20000) * 1.1e6
    for policy, m in (("recent", 10), ("uniform", 10), ("uniform", 25), ("uniform", 300)):
        i1, c1 = batch_find_arrays(g, qv, qt, m, policy=policy, seed=31)
        i2, c2 = ofinder.batch_find_arrays(og, qv, qt, m, policy=policy, seed=31)
        np.testing.assert_array_equal(i1, i2)
        np.testing.assert_array_equal(c1, c2)


@pytest.mark.parametrize("p,m", [(20, 10), (9, 6), (12, 11), (300, 25)])
def test_device_uniform_marginals_chi_square(p, m):
    """Each valid entry appears with frequency m/p (test_finder.py:79-95)."""
    from scipy import stats
    from paper_2402_05396_b200 import batch_find_arrays, build_graph
    g = build_graph([0] * p, list(range(1, p + 1)), list(np.arange(1.0, p + 1.0)), num_nodes=p + 1)
    trials = 200_000
    idx, cnt = batch_find_arrays(g, np.zeros(trials, np.int64), np.full(trials, float(p + 1)), m,
                                 policy="uniform", seed=777)
    assert (cnt == m).all()
    local = idx - int(_np(g.tcsr_offsets)[0])
    counts = np.bincount(local.ravel(), minlength=p).astype(float)
    expected = trials * m / p
    chi2 = ((counts - expected) ** 2 / expected).sum()
    assert chi2 < stats.chi2.ppf(1 - 1e-3, df=p - 1)
    assert all(len(set(r.tolist())) == m for r in idx[:2000])


def test_device_finder_validation():
    from paper_2402_05396_b200 import batch_find, batch_find_arrays, build_graph
    from paper_2402_05396_b200.finder import NeighborQuery
    g = build_graph([0, 1], [1, 2], [1.0, 2.0])
    with pytest.raises(ValueError):
        batch_find_arrays(g, [0, 1], [1.0], 3)
    with pytest.raises(ValueError):
        batch_find_arrays(g, [0], [1.0], 0)
    with pytest.raises(ValueError):
        batch_find_arrays(g, [0], [1.0], 2, policy="bogus")
    with pytest.raises(ValueError):
        batch_find(g, [NeighborQuery(0, 1.0, 2), NeighborQuery(0, 1.0, 3)])
    nb = batch_find(g, [NeighborQuery(1, 5.0, 3)])[0]
    assert list(nb.ts) == [2.0, 1.0] and list(nb.nodes) == [2, 0]


# ---------------------------------------------------------------- K5/K6 cache
def test_device_cache_bit_exact():
    from paper_2402_05396_b200 import cache as dcache
    z = load_golden("cache")
    for ci in range(5):
        k, eps = int(z[f"c{ci}/k"]), int(z[f"c{ci}/eps"])
        E = z[f"c{ci}/e0/counters"].shape[0]
        st = dcache.make_cache(E, k, epsilon=eps)
        for ep in range(int(z[f"c{ci}/epochs"])):
            _, hits = dcache.lookup(st, z[f"c{ci}/e{ep}/eids"])
            np.testing.assert_array_equal(hits, z[f"c{ci}/e{ep}/hits"])
            np.testing.assert_array_equal(_np(st.counters), z[f"c{ci}/e{ep}/counters"])
            assert [st.epoch_stats[-1].hits, st.epoch_stats[-1].misses] == list(z[f"c{ci}/e{ep}/hm"])
            assert dcache.maybe_replace(st) == bool(z[f"c{ci}/e{ep}/replaced"])
            np.testing.assert_array_equal(_np(st.resident), z[f"c{ci}/e{ep}/resident"])
            assert (_np(st.counters) == 0).all()


def test_device_oracle_cache_rates():
    from paper_2402_05396_b200 import oracle_cache
    z = load_golden("cache")
    for k in (0, 1, 7, 30, 80):
        r = oracle_cache(z["oracle/counts"], k)
        np.testing.assert_array_equal(np.array([np.nan if x is None else x for x in r]), z[f"oracle/k{k}"])


def test_device_cache_replace_large_vs_oracle():
    """Radix select over 3M counters with heavy ties at the k-th key."""
    import torch
    from oracle.cache import OracleCache
    from paper_2402_05396_b200 import cache as dcache
    rng = np.random.default_rng(5)
    E = 3_000_000
    ost = OracleCache(E, 0.2)
    dst_ = dcache.make_cache(E, 0.2)
    for ep in range(3):
        eids = np.minimum(rng.zipf(1.1, 2_000_000) - 1, E - 1)
        _, h1 = ost.lookup(eids)
        _, h2 = dcache.lookup(dst_, torch.as_tensor(eids).cuda())
        assert np.array_equal(h1, _np(h2))
        assert ost.maybe_replace() == dcache.maybe_replace(dst_)
        np.testing.assert_array_equal(ost.resident, _np(dst_.resident))
        assert ost.epochs[-2] == [dst_.epoch_stats[-2].hits, dst_.epoch_stats[-2].misses]


def test_device_lookup_index_error_and_features():
    from paper_2402_05396_b200 import cache as dcache
    feats = np.random.default_rng(0).normal(size=(10, 4)).astype(np.float32)
    st = dcache.make_cache(10, k=2, features=feats)
    with pytest.raises(IndexError):
        dcache.lookup(st, [10])
    got, hits = dcache.lookup(st, [3, 7])
    np.testing.assert_array_equal(got, feats[[3, 7]])
    assert hits.tolist() == [False, False]


def test_device_hot_tier_serves_identical_rows():
    """A physical hot tier (rows copied into a dense [k, d] block) changes no value."""
    import torch
    from paper_2402_05396_b200 import cache as dcache
    from paper_2402_05396_b200.graph import feat_store
    from paper_2402_05396_b200 import _lib
    rng = np.random.default_rng(1)
    feats = torch.as_tensor(rng.normal(size=(5000, 172)).astype(np.float32)).cuda()
    st = dcache.make_cache(5000, 0.1, features=feats, hot_tier=True)
    dcache.lookup(st, torch.as_tensor(np.minimum(rng.zipf(1.2, 20000) - 1, 4999)).cuda())
    assert dcache.maybe_replace(st)
    ids = torch.as_tensor(rng.integers(0, 5000, 3000)).cuda()
    mask = torch.as_tensor(rng.random(3000) < 0.7).cuda()
    out = torch.empty((3000, 172), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib.tg_lookup_gather(_lib.ptr(ids), _lib.ptr(mask), 3000, st.c_store(), st.c_cache(), 0,
                                         _lib.ptr(out), 172, _lib.stream_ptr()))
    exp = torch.where(mask[:, None], feats[ids], torch.zeros((), device="cuda"))
    assert torch.equal(out.view(torch.int32), exp.view(torch.int32))
    assert int((st.slot_of >= 0).sum()) == st.k


def test_device_node_rows_signed_zeros():
    """_node_feature_rows(ids, mask) == rows * mask (training.py:227-229)."""
    import torch
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.graph import feat_store
    rng = np.random.default_rng(2)
    nf = rng.normal(size=(50, 100)).astype(np.float32)
    ids = rng.integers(0, 50, (64, 10))
    mask = rng.random((64, 10)) < 0.6
    ids[~mask] = 0
    nft = torch.as_tensor(nf).cuda()
    out = torch.empty((640, 100), dtype=torch.float32, device="cuda")
    idt, mt = torch.as_tensor(ids).cuda(), torch.as_tensor(mask).cuda()
    _lib.check(_lib.lib.tg_lookup_gather(_lib.ptr(idt), _lib.ptr(mt), 640, feat_store(nft), None, 1, _lib.ptr(out),
                                         100, _lib.stream_ptr()))
    exp = (nf[ids].astype(np.float64) * mask[..., None].astype(np.float64)).reshape(640, 100)
    assert _np(out).astype(np.float64).tobytes() == exp.tobytes()


# ---------------------------------------------------------------- K8 WOR
@pytest.mark.parametrize("ci", range(5))
def test_device_wor_bit_exact_given_reference_q(ci):
    from paper_2402_05396_b200.sampler import PolicyOutput, sample_without_replacement
    from oracle.wor import sample_wor
    z = load_golden("wor")
    n = int(z[f"w{ci}/n"])
    rng = np.random.default_rng(int(z[f"w{ci}/seed"]))
    pol = PolicyOutput(q=z[f"w{ci}/q"], log_q=z[f"w{ci}/log_q"], mask=z[f"w{ci}/mask"])
    sample_without_replacement(pol, n, rng)
    np.testing.assert_array_equal(pol.selected, z[f"w{ci}/selected"])
    np.testing.assert_array_equal(pol.selected_mask, z[f"w{ci}/selected_mask"])
    assert pol.selected_log_q.tobytes() == z[f"w{ci}/selected_log_q"].tobytes()
    # the generator is left where the reference leaves it
    rng2 = np.random.default_rng(int(z[f"w{ci}/seed"]))
    sample_wor(z[f"w{ci}/q"], z[f"w{ci}/log_q"], n, rng2)
    assert rng.random() == rng2.random()


def test_device_wor_large_batch_vs_oracle():
    import torch
    from paper_2402_05396_b200.sampler import sample_wor_device
    from oracle.wor import sample_wor
    rng = np.random.default_rng(3)
    B, m, n = 12000, 25, 10
    mask = rng.random((B, m)) < 0.85
    logits = rng.normal(size=(B, m)) * 2
    e = np.where(mask, np.exp(logits - logits.max(1, keepdims=True)), 0.0)
    z = e.sum(1, keepdims=True)
    q = np.divide(e, z, out=np.zeros_like(e), where=z > 0)
    lq = np.where(mask, np.log(np.maximum(q, 1e-300)), -1e30)
    sel, sm, slq = sample_wor_device(torch.as_tensor(q).cuda(), torch.as_tensor(lq).cuda(), n,
                                     np.random.default_rng(99))
    s2, m2, l2 = sample_wor(q, lq, n, np.random.default_rng(99))
    np.testing.assert_array_equal(_np(sel), s2)
    np.testing.assert_array_equal(_np(sm), m2)
    assert _np(slq).tobytes() == l2.tobytes()


# ---------------------------------------------------------------- whole batches
def _pipeline(tag):
    from test_oracle_golden import _pipeline_cfg, _pipeline_spec
    return _pipeline_spec(tag), _pipeline_cfg(tag)


@pytest.mark.parametrize("tag", ["A", "B", "E", "Bv"])
def test_device_pipeline_matches_reference_trainer(tag):
    """Fused find+materialise+expand+cache+gather equals the reference
    Trainer's mini-batches over two epochs (golden digests of f64 buffers)."""
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    z = load_golden("pipeline")
    V, E, d_e, d_v, gseed, tseed, iters = (int(x) for x in z[f"{tag}/meta"])
    spec, cfg = _pipeline(tag)
    og = oshapes.make_graph(spec, seed=gseed)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                    edge_features=og.edge_features)
    gen = MiniBatchGenerator(g, cfg, seed=tseed)
    assert gen.iters_per_epoch == iters
    for ep in range(2):
        for it in z[f"{tag}/its"]:
            p = f"{tag}/ep{ep}/it{it}"
            nodes, times = gen.roots_for_iteration(int(it))
            np.testing.assert_array_equal(nodes, z[p + "/nodes"])
            recs = gen.generate(torch.as_tensor(nodes).cuda(), torch.as_tensor(times).cuda(), int(it))
            for rec in recs:
                l = rec["layer"]
                for k in ("sel_ids", "sel_eids", "sel_mask"):
                    np.testing.assert_array_equal(_np(rec[k]), z[f"{p}/l{l}/{k}"], err_msg=f"{p} l{l} {k}")
                assert _np(rec["sel_dts"]).tobytes() == z[f"{p}/l{l}/sel_dts"].tobytes()
                for k in ("edge_rows", "node_rows", "tgt_rows"):
                    if f"{p}/l{l}/{k}_sha" in z:
                        got = _np(rec[k]).astype(np.float64)
                        np.testing.assert_array_equal(_sha(got), z[f"{p}/l{l}/{k}_sha"], err_msg=f"{p} l{l} {k}")
            if gen.cache is not None:
                np.testing.assert_array_equal(_np(gen.cache.counters), z[p + "/counters"])
        if gen.cache is not None:
            st = gen.cache.epoch_stats[-1]
            assert [st.hits, st.misses] == list(z[f"{tag}/ep{ep}/hm"])
            assert gen.end_epoch() == bool(z[f"{tag}/ep{ep}/replaced"])
            np.testing.assert_array_equal(_np(gen.cache.resident), z[f"{tag}/ep{ep}/resident"])


def test_device_pipeline_gdelt_slice_vs_oracle():
    """GDELT-shaped (V=16,682, d_e=186) at 2M events, batch 600, 2-hop recent:
    full-width device batches bit-exact against the oracle for 3 iterations."""
    import torch
    from oracle import shapes as oshapes
    from oracle.pipeline import OracleMiniBatch
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["E"].scaled(2_000_000 / SHAPES["E"].E)
    og = oshapes.make_graph(spec, seed=1)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = spec.path_config()
    gen = MiniBatchGenerator(g, cfg, seed=0)
    ob = OracleMiniBatch(og, cfg, seed=0, dtype=np.float32)
    for it in (5, gen.iters_per_epoch // 2, gen.iters_per_epoch - 1):
        nodes, times = ob.roots_for_iteration(it)
        recs = gen.generate(torch.as_tensor(nodes).cuda(), torch.as_tensor(times).cuda(), it)
        for r, o in zip(recs, ob.generate(nodes, times, it)):
            for k in ("sel_ids", "sel_eids", "sel_mask", "sel_dts", "edge_rows"):
                assert _np(r[k]).tobytes() == o[k].astype(_np(r[k]).dtype).tobytes(), (it, r["layer"], k)
            if "next_v" in r:
                assert _np(r["next_v"]).tobytes() == o["next_v"].tobytes()
                assert _np(r["next_t"]).tobytes() == o["next_t"].tobytes()
    np.testing.assert_array_equal(_np(gen.cache.counters), ob.cache.counters)


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


# ---------------------------------------------------------------- K7 scoring
def _score_case(tag, precision):
    import torch
    from test_oracle_golden import scoring_inputs
    from paper_2402_05396_b200.params import ScoringModel, sampler_params
    from paper_2402_05396_b200.scoring import score_policy
    z = load_golden("scoring")
    c = scoring_inputs(z, tag)
    p = sampler_params(c["store_seed"], c["enc"], c["m"], c["d_v"], c["d_e"], c["decoder"])
    model = ScoringModel(p, c["decoder"], c["enc"], c["m"], c["d_v"], c["d_e"], c["alpha"], c["beta"],
                         precision=precision)
    dev = lambda x, dt: None if x is None else torch.as_tensor(x).to("cuda", dt)  # noqa: E731
    q, lq = score_policy(model, dev(c["ids"], torch.int64), dev(c["dts"], torch.float64), dev(c["mask"], torch.bool),
                         dev(c["node_rows"], torch.float32), dev(c["edge_rows"], torch.float32),
                         dev(c["tgt_rows"], torch.float32))
    return _np(q).astype(np.float64), _np(lq).astype(np.float64), z[f"{tag}/q"], z[f"{tag}/log_q"], c["mask"]


SCORE_TAGS = ["s0", "s1", "s2", "s3", "s4", "s5", "s6", "s7"]


@pytest.mark.parametrize("tag", SCORE_TAGS)
def test_device_scoring_f32_within_1e5(tag):
    """f32 device policy (q, log q) within 1e-5 relative of the reference's
    float64 policy (north-star tolerance); masked slots exact."""
    q, lq, rq, rlq, mask = _score_case(tag, "float32")
    assert np.all(q[~mask] == 0.0) and np.all(lq[~mask] == np.float64(np.float32(-1e30)))
    assert np.all(np.abs(q - rq) <= 1e-5 * np.abs(rq) + 1e-12), np.max(np.abs(q - rq) / np.maximum(rq, 1e-30))
    assert np.all(np.abs(lq - rlq) <= 1e-5 * np.maximum(np.abs(rlq), 1.0))


@pytest.mark.parametrize("variant", ["TG_K7_TOKMIX_TC", "TG_K7_TOKMIX_BLK", "TG_K7_TOKMIX_WARP"])
@pytest.mark.parametrize("tag", ["s4", "s5", "s6", "s7"])
def test_device_scoring_f32_token_mixer_variants(tag, variant, monkeypatch):
    """The m = 25 cases through the opt-in token mixers (channel blocks,
    warp per root): within 1e-5 of the reference like the default CTA
    kernel, and within 2e-6 of it."""
    q0, lq0, rq, rlq, mask = _score_case(tag, "float32")
    monkeypatch.setenv(variant, "1")
    q, lq, _, _, _ = _score_case(tag, "float32")
    assert np.all(np.abs(q - rq) <= 1e-5 * np.abs(rq) + 1e-12)
    assert np.all(np.abs(lq - rlq) <= 1e-5 * np.maximum(np.abs(rlq), 1.0))
    assert np.all(np.abs(q - q0) <= 2e-6 * np.abs(q0) + 1e-12)


@pytest.mark.parametrize("tag", SCORE_TAGS)
def test_device_scoring_f64_matches_reference(tag):
    """f64 device policy equals the reference's to float64 rounding."""
    q, lq, rq, rlq, mask = _score_case(tag, "float64")
    np.testing.assert_allclose(q, rq, rtol=1e-11, atol=1e-300)
    np.testing.assert_allclose(lq, rlq, rtol=1e-11, atol=1e-11)


def _adaptive_run(tag, precision):
    import torch
    from test_oracle_golden import adaptive_setup
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    z, spec, cfg, gseed, tseed, iters = adaptive_setup(tag)
    cfg.precision = precision
    og = oshapes.make_graph(spec, seed=gseed)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                    edge_features=og.edge_features)
    gen = MiniBatchGenerator(g, cfg, seed=tseed)
    assert gen.iters_per_epoch == iters
    out = []
    for it in z[f"{tag}/its"]:
        nodes, times = gen.roots_for_iteration(int(it))
        recs = gen.generate(torch.as_tensor(nodes).cuda(), torch.as_tensor(times).cuda(), int(it))
        out.append((int(it), [{k: (_np(v) if hasattr(v, "detach") else v) for k, v in r.items()
                               if k not in ("queries",)} for r in recs], _np(gen.cache.counters)))
    return z, out


@pytest.mark.parametrize("tag", ["C", "D", "Dt", "Cg"])
def test_device_adaptive_pipeline_f64_matches_reference_trainer(tag):
    """Adaptive layers end to end in float64 (the reference's default
    precision): selections, selected rows, PP edge rows and cache counters
    bit-exact against the reference Trainer; q to f64 rounding."""
    z, out = _adaptive_run(tag, "float64")
    for it, recs, counters in out:
        p = f"{tag}/it{it}"
        for r in recs:
            l = r["layer"]
            np.testing.assert_allclose(r["q"], z[f"{p}/l{l}/q"], rtol=1e-10, atol=1e-300)
            np.testing.assert_array_equal(r["selected"], z[f"{p}/l{l}/selected"])
            for k in ("sel_ids", "sel_eids", "sel_mask"):
                np.testing.assert_array_equal(r[k], z[f"{p}/l{l}/{k}"], err_msg=f"{p} l{l} {k}")
            assert r["sel_dts"].tobytes() == z[f"{p}/l{l}/sel_dts"].tobytes()
            for k in ("edge_rows", "node_rows", "tgt_rows"):
                if f"{p}/l{l}/{k}_sha" in z:
                    np.testing.assert_array_equal(_sha(r[k].astype(np.float64)), z[f"{p}/l{l}/{k}_sha"],
                                                  err_msg=f"{p} l{l} {k}")
        np.testing.assert_array_equal(counters, z[p + "/counters"])


@pytest.mark.parametrize("tag", ["C", "D"])
def test_device_adaptive_pipeline_f32(tag):
    """float32 fast mode: q within 1e-5 of the reference; the selection may
    differ only where a draw lands within the f32 error of a cumsum
    boundary, so >= 99% of rows match exactly and every row is valid."""
    z, out = _adaptive_run(tag, "float32")
    for it, recs, counters in out:
        p = f"{tag}/it{it}"
        for r in recs:
            l = r["layer"]
            rq = z[f"{p}/l{l}/q"]
            assert np.all(np.abs(r["q"] - rq) <= 1e-5 * rq + 1e-12)
            sel, ref = r["selected"], z[f"{p}/l{l}/selected"]
            same = np.all(sel == ref, axis=1)
            assert same.mean() >= 0.99, same.mean()
            cm = z[f"{p}/l{l}/cand_mask"]
            for b in np.flatnonzero(~same):
                s = sel[b][sel[b] >= 0]
                assert np.all(cm[b][s]) and np.all(np.diff(s) > 0)


# ---------------------------------------------------------------- K9 root sharding
@pytest.mark.parametrize("tag,world", [("B", 2), ("E", 3), ("D", 2)])
def test_device_root_shards_reassemble_bit_exact(tag, world):
    """Each rank's block of roots, generated with its global row keys
    (shard.layer_rows -> tg_rowmap / WOR position), reassembles into the
    single-GPU mini-batch bit for bit; summed cache counters agree."""
    import torch
    from test_shard_gloo import CASES, _reassemble
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES
    from paper_2402_05396_b200.shard import layer_rows, root_partition
    key, f, kw, batch = CASES[tag]
    spec = SHAPES[key].scaled(f)
    cfg = PathConfig(batch_size=batch, cache_fraction=0.2, **kw)
    og = oshapes.make_graph(spec, seed=3)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                    edge_features=og.edge_features)
    full = MiniBatchGenerator(g, cfg, seed=1)
    parts = [MiniBatchGenerator(g, cfg, seed=1) for _ in range(world)]
    for it in (0, full.iters_per_epoch // 2, full.iters_per_epoch - 1):
        nodes, times = full.roots_for_iteration(it)
        R1 = nodes.shape[0]
        ref = [{k: _np(v) for k, v in r.items() if k in ("sel_ids", "sel_eids", "sel_dts", "sel_mask", "edge_rows")}
               for r in full.generate(torch.as_tensor(nodes).cuda(), torch.as_tensor(times).cuda(), it)]
        outs = []
        for rank, gen in enumerate(parts):
            a, b = root_partition(R1, rank, world)
            lrs = layer_rows(R1, cfg.n, a, b, gen.L)
            recs = gen.generate(torch.as_tensor(nodes[a:b]).cuda(), torch.as_tensor(times[a:b]).cuda(), it,
                                layer_rows=lrs)
            outs.append([{k: _np(v) for k, v in r.items() if k in ref[0]} for r in recs])
        for li, r in enumerate(ref):
            for k, v in r.items():
                got = _reassemble([outs[rank][li][k] for rank in range(world)], R1, cfg.n, world, li)
                assert got.tobytes() == np.ascontiguousarray(v).tobytes(), (tag, it, li, k)
    total = sum(_np(p.cache.counters) for p in parts)
    np.testing.assert_array_equal(total, _np(full.cache.counters))


def test_device_inflight_slots_match_sequential():
    """Batches generated on two in-flight slots (own buffers + streams)
    equal the sequential results, and the cache counters agree."""
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["E"].scaled(0.0002)
    og = oshapes.make_graph(spec, seed=2)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = PathConfig(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=False, n=10, batch_size=128)
    seq, par = MiniBatchGenerator(g, cfg, seed=0), MiniBatchGenerator(g, cfg, seed=0)
    its = list(range(0, seq.iters_per_epoch, max(1, seq.iters_per_epoch // 6)))[:6]
    roots = [tuple(torch.as_tensor(x).cuda() for x in seq.roots_for_iteration(it)) for it in its]
    ref = []
    for (n, t), it in zip(roots, its):
        ref.append([{k: _np(r[k]) for k in ("sel_ids", "sel_dts", "edge_rows")} for r in seq.generate(n, t, it)])
    outs = []
    main = torch.cuda.current_stream()
    for k in (1,):
        par.slot_stream(k).wait_stream(main)
    for i, ((n, t), it) in enumerate(zip(roots, its)):
        recs = par.generate(n, t, it, slot=i % 2)
        par.join()
        outs.append([{k: _np(r[k]) for k in ("sel_ids", "sel_dts", "edge_rows")} for r in recs])
    for a, b in zip(ref, outs):
        for ra, rb in zip(a, b):
            for k in ra:
                assert ra[k].tobytes() == rb[k].tobytes()
    np.testing.assert_array_equal(_np(seq.cache.counters), _np(par.cache.counters))


# ---------------------------------------------------------------- K7 tensor-core GEMM
@pytest.mark.parametrize("M,K,N", [(128, 8, 16), (300, 325, 325), (1000, 266, 100), (257, 425, 425), (64, 172, 100)])
def test_device_tc_gemm_3xtf32_matches_fp64(M, K, N):
    """tcgen05 3xTF32 GEMM (UTCHMMA, TMEM accumulate) equals the fp64
    product to ~fp32 accuracy: |err| <= 2e-6 * sum_k |a_k b_k|."""
    import ctypes
    import torch
    from paper_2402_05396_b200 import _lib
    g = torch.Generator().manual_seed(M * 7 + K)
    lda = (K + 3) // 4 * 4
    A = torch.zeros(M, lda, dtype=torch.float32)
    A[:, :K] = torch.randn(M, K, generator=g)
    W = torch.randn(K, N, generator=g) / K ** 0.5
    bias = torch.randn(N, generator=g)
    ref = A[:, :K].double() @ W.double() + bias.double()
    scale = A[:, :K].double().abs() @ W.double().abs() + bias.double().abs()
    Ad, Wd, bd = A.cuda(), W.cuda(), bias.cuda()
    C = torch.full((M, N), float("nan"), device="cuda")
    nb = ctypes.c_size_t(0)
    _lib.check(_lib.lib.tg_tc_gemm_workspace(M, N, K, ctypes.byref(nb)))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib.tg_tc_gemm(_lib.ptr(Ad), lda, M, K, _lib.ptr(Wd), N, N, _lib.ptr(bd), _lib.ptr(C), N,
                                   _lib.ptr(ws), _lib.stream_ptr()))
    err = (C.cpu().double() - ref).abs()
    assert torch.isfinite(C).all()
    assert (err <= 2e-6 * scale + 1e-30).all(), float((err / scale).max())


@pytest.mark.parametrize("env", [{"TG_TC_PACKA": "1"}, {"TG_TC_CLUSTER": "1"}, {"TG_TC_NO_CLUSTER": "1"},
                                 {"TG_TC_PACKA": "1", "TG_TC_NO_CLUSTER": "1"}, {"TG_TC_PAIR": "1"}])
def test_device_tc_gemm_variants(env):
    """The other K7 GEMM feeds (pre-split A image, 2-CTA weight multicast,
    independent CTAs, cta_group::2 CTA pairs) pass the GEMM and scoring parity tests too (the switches
    are read once per process, hence the subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k",
                        "tc_gemm_3xtf32 or scoring or graphmixer", "-p", "no:cacheprovider",
                        os.path.join(root, "tests")], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# ---------------------------------------------------------------- sharded placement
@pytest.mark.parametrize("world,register", [(1, False), (3, False), (4, True)])
def test_device_sharded_table_generator_bit_exact(world, register, monkeypatch):
    """Edge rows served from a row-range-sharded table (peer pointer table,
    replicated hot tier after an epoch boundary) equal the dense-table
    mini-batch bit for bit, on both K5 paths; cache counters agree."""
    import dataclasses
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.placement import ShardedTable
    from paper_2402_05396_b200.shapes import SHAPES
    if register:
        monkeypatch.setenv("TG_K5_REGISTER_PATH", "1")
    spec = SHAPES["E"].scaled(0.0003)
    og = oshapes.make_graph(spec, seed=4)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    gs = dataclasses.replace(g, edge_features=ShardedTable.split_local(g.edge_features, world))
    for kw in (dict(aggregator="tgat", finder_policy="recent", adaptive_neighbor=False),
               dict(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=False)):
        cfg = PathConfig(n=10, batch_size=100, cache_fraction=0.2, **kw)
        dense, shard = MiniBatchGenerator(g, cfg, seed=0), MiniBatchGenerator(gs, cfg, seed=0)
        assert shard.cache.hot is not None
        its = [0, dense.iters_per_epoch // 3, dense.iters_per_epoch - 1]
        for epoch in range(2):
            for it in its:
                n, t = (torch.as_tensor(x).cuda() for x in dense.roots_for_iteration(it))
                a = [{k: _np(r[k]) for k in ("sel_eids", "sel_mask", "edge_rows")} for r in dense.generate(n, t, it)]
                b = [{k: _np(r[k]) for k in ("sel_eids", "sel_mask", "edge_rows")} for r in shard.generate(n, t, it)]
                for ra, rb in zip(a, b):
                    for k in ra:
                        assert ra[k].tobytes() == rb[k].tobytes(), (world, epoch, it, k)
            np.testing.assert_array_equal(_np(dense.cache.counters), _np(shard.cache.counters))
            assert dense.end_epoch() == shard.end_epoch()
        assert shard.cache.resident_count > 0


def test_device_sharded_table_lookup_and_adaptive():
    """cache.lookup and the adaptive layer's candidate rows through a
    sharded table equal the dense results."""
    import dataclasses
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200 import cache as dcache
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.placement import ShardedTable, shard_bounds
    from paper_2402_05396_b200.shapes import SHAPES
    rng = np.random.default_rng(3)
    feats = torch.as_tensor(rng.normal(size=(7001, 172)).astype(np.float32)).cuda()
    st = dcache.make_cache(7001, 0.1, features=ShardedTable.split_local(feats, 5))
    ids = torch.as_tensor(rng.integers(0, 7001, 4000)).cuda()
    out, hits = dcache.lookup(st, ids)
    assert torch.equal(out.view(torch.int32), feats[ids].view(torch.int32))
    assert shard_bounds(7001, 4, 5) == (5604, 7001, 1401)
    spec = SHAPES["D"].scaled(0.001)
    og = oshapes.make_graph(spec, seed=5)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                    edge_features=og.edge_features)
    gs = dataclasses.replace(g, edge_features=ShardedTable.split_local(g.edge_features, 2))
    cfg = PathConfig(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=True, decoder="gatv2", m=12,
                     n=5, batch_size=16, precision="float32")
    dense, shard = MiniBatchGenerator(g, cfg, seed=1), MiniBatchGenerator(gs, cfg, seed=1)
    it = dense.iters_per_epoch // 2
    n, t = (torch.as_tensor(x).cuda() for x in dense.roots_for_iteration(it))
    for ra, rb in zip(dense.generate(n, t, it), shard.generate(n, t, it)):
        for k in ("sel_eids", "edge_rows", "cand_edge_rows", "q"):
            if k in ra:
                assert _np(ra[k]).tobytes() == _np(rb[k]).tobytes(), k


def test_device_sharded_table_ipc_two_processes():
    """Two processes on cuda:0 (gloo for the handle exchange) each own one
    shard, map the other's through CUDA IPC, and gather rows of both shards
    bit-exactly (tests/mp_sharded_worker.py)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(here, "mp_sharded_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("sharded-ipc ok") == 2, r.stdout[-2000:]


def test_device_fmat_load_into_pitched_table(tmp_path):
    """load_features_device == load_features (f32 and f64 files), rows
    landing in the 16-B-pitched table; chunked staging across many chunks."""
    import os
    import torch
    from conftest import GOLDEN
    from paper_2402_05396_b200 import matio
    from paper_2402_05396_b200.graph import row_pitch
    for name in ("feat_f32.fmat", "feat_f64.fmat"):
        path = os.path.join(GOLDEN, name)
        exp = matio.load_features(path)
        got = matio.load_features_device(path, chunk_bytes=64)
        assert got.stride(0) == row_pitch(exp.shape[1])
        assert _np(got).tobytes() == exp.tobytes()
    big = np.random.default_rng(0).normal(size=(100_003, 186)).astype(np.float32)
    matio.save_features(tmp_path / "big.fmat", big)
    got = matio.load_features_device(tmp_path / "big.fmat", chunk_bytes=1 << 20)
    assert torch.equal(got.cpu(), torch.as_tensor(big))


# ---------------------------------------------------------------- ingest
@pytest.mark.parametrize("name", ["crlf.csv", "cr.csv", "plain.csv", "wide.csv"])
def test_device_ingest_matches_reference(name):
    import os
    from conftest import GOLDEN
    from paper_2402_05396_b200.ingest import ingest_events
    z = load_golden("ingest")
    g = ingest_events(os.path.join(GOLDEN, "ingest", name))
    np.testing.assert_array_equal(_np(g.src), z[f"{name}/src"])
    np.testing.assert_array_equal(_np(g.dst), z[f"{name}/dst"])
    assert _np(g.ts).tobytes() == z[f"{name}/ts"].tobytes()
    np.testing.assert_array_equal(_np(g.tcsr_offsets), z[f"{name}/offsets"])
    if f"{name}/ef" in z:
        ef, ref = _np(g.edge_features), z[f"{name}/ef"]
        same = (ef.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(ef) & np.isnan(ref))
        assert same.all()


@pytest.mark.parametrize("name", ["err_few.csv", "err_int.csv", "err_float.csv", "err_nonfinite.csv",
                                  "err_width.csv"])
def test_device_ingest_errors_match_reference(name):
    import os
    from conftest import GOLDEN
    from paper_2402_05396_b200 import DataError
    from paper_2402_05396_b200.ingest import ingest_events
    z = load_golden("ingest")
    d = os.path.join(GOLDEN, "ingest")
    with pytest.raises(DataError) as exc:
        ingest_events(os.path.join(d, name))
    assert str(exc.value).replace(d + "/", "") == str(z[f"{name}/error"])


def test_device_manifest_dataset_matches_reference():
    """A dataset written by the reference's save_dataset (repr floats, FMAT
    node features) loads to the same device graph."""
    import os
    from conftest import GOLDEN
    from paper_2402_05396_b200.ingest import load_manifest
    z = load_golden("ingest")
    g = load_manifest(os.path.join(GOLDEN, "ingest", "ds.manifest.json"))
    for k in ("src", "dst", "tcsr_offsets", "tcsr_neighbors", "tcsr_eids"):
        np.testing.assert_array_equal(_np(getattr(g, k)), z[f"ds/{k}"])
    for k in ("ts", "tcsr_ts", "edge_features", "node_features"):
        assert _np(getattr(g, k)).tobytes() == z[f"ds/{k}"].tobytes(), k


def test_device_ingest_large_vs_oracle(tmp_path):
    """200k repr-formatted lines with 20 f32 features: device parse == the
    oracle's per-line Python parse, bit for bit."""
    from oracle import ingest as oing
    from paper_2402_05396_b200.ingest import ingest_arrays_device
    r = np.random.default_rng(5)
    n = 200_000
    src = r.integers(0, 5000, n)
    dst = r.integers(0, 5000, n)
    ts = np.sort(r.random(n) * 1e7)
    f = r.normal(size=(n, 20)).astype(np.float32) * np.float32(10.0) ** r.integers(-8, 8, (n, 20)).astype(np.float32)
    path = tmp_path / "big.csv"
    with open(path, "w") as fh:
        for i in range(n):
            fh.write(f"{src[i]},{dst[i]},{float(ts[i])!r}," + ",".join(repr(float(x)) for x in f[i]) + "\n")
    es, ed, et, ef = oing.ingest_arrays(path)
    ds, dd, dt, df = ingest_arrays_device(path)
    np.testing.assert_array_equal(_np(ds), es)
    np.testing.assert_array_equal(_np(dd), ed)
    assert _np(dt).tobytes() == et.tobytes()
    assert _np(df).tobytes() == ef.tobytes()


def test_device_ingest_long_decimals_parsed_like_python(tmp_path):
    """Values of > 19 significant digits whose rounding the device cannot
    settle (exact halfway points plus a tail) are re-parsed on the host with
    Python's float(), like graph.py:170-179 -- the file loads, bit-exact."""
    from oracle import ingest as oing
    from paper_2402_05396_b200 import DataError
    from paper_2402_05396_b200.ingest import ingest_arrays_device
    half = "1.00000000000000011102230246251565404236316680908203125"  # 1 + 2^-53: ties to 1.0
    above = half[:-1] + "6"                                           # just above: 1 + 2^-52
    lines = [f"{i % 7},{(i * 3) % 11},{float(i)!r},0.5,{half if i % 3 else above}" for i in range(3000)]
    lines[17] = f"1,2,{above},{half},{above}"
    lines[2500] = f"3,4,2500{half[1:]},{above},0.25"
    path = tmp_path / "long.csv"
    path.write_text("\n".join(lines) + "\n")
    es, ed, et, ef = oing.ingest_arrays(path)
    ds, dd, dt, df = ingest_arrays_device(path)
    np.testing.assert_array_equal(_np(ds), es)
    np.testing.assert_array_equal(_np(dd), ed)
    assert _np(dt).tobytes() == et.tobytes()
    assert _np(df).tobytes() == ef.tobytes()
    assert float(half) == 1.0 and float(above) > 1.0
    # a genuine error after such lines is still reported at its own line
    lines[2900] = "5,6,notanumber,1,2"
    path.write_text("\n".join(lines) + "\n")
    with pytest.raises(DataError, match=":2901: could not convert"):
        ingest_arrays_device(path)
    # and a long decimal that is non-finite for Python is the first error
    lines[40] = "1,2," + "9" * 400 + ",1,2"
    path.write_text("\n".join(lines) + "\n")
    with pytest.raises(DataError, match=":41: non-finite timestamp"):
        ingest_arrays_device(path)
