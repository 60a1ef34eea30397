"""The reference's own test cases, run against the drop-in API on the GPU.

Restatements (same inputs, same assertions, written against this package's
names) of the cases in the reference's test suite that pin results at the
mini-batch-generation boundary:

  pkg/tests/test_finder.py:19-167    pivots, recency, uniformity, batch API
  pkg/tests/test_cache.py             lookup, replacement, oracle, report
  pkg/tests/test_sampler.py:22-212    mixer_transform, decoders, WOR sampling
  pkg/tests/test_encoders.py          masked rows, widths, target embedding

Gradient checks that the reference runs with finite differences on its
autodiff (test_sampler.py:75-84, 141-155) are run here on the device
backward (tg_score_backward) against finite differences of the device
forward (tg_score, f64)."""

import json

import numpy as np
import pytest
from scipy import stats

pytestmark = pytest.mark.gpu


def _np(x):
    import torch
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)


def chain_graph(ts_list):
    from paper_2402_05396_b200 import build_graph
    k = len(ts_list)
    return build_graph([0] * k, list(range(1, k + 1)), ts_list, num_nodes=k + 1)


def random_graph(rng, num_nodes=50, num_events=400, d_v=0, d_e=0):
    from paper_2402_05396_b200 import build_graph
    src = rng.integers(0, num_nodes, num_events)
    dst = rng.integers(0, num_nodes, num_events)
    ts = np.sort(rng.random(num_events) * 100.0)
    nf = rng.normal(size=(num_nodes, d_v)).astype(np.float32) if d_v else None
    ef = rng.normal(size=(num_events, d_e)).astype(np.float32) if d_e else None
    return build_graph(src, dst, ts, num_nodes=num_nodes, node_features=nf, edge_features=ef)


def adjacency(g, v):
    nbr, ts, eids = g.adjacency(v)
    return _np(nbr), _np(ts), _np(eids)


# ---------------------------------------------------------------- finder (test_finder.py)
class TestPivot:
    def test_strict_less_with_ties(self):
        from paper_2402_05396_b200 import pivot
        assert pivot(chain_graph([1.0, 3.0, 3.0, 7.0]), 0, 3.0) == 1

    def test_time_beyond_all(self):
        from paper_2402_05396_b200 import pivot
        assert pivot(chain_graph([1.0, 3.0, 3.0, 7.0]), 0, 100.0) == 4

    def test_matches_linear_scan(self, rng):
        from paper_2402_05396_b200 import pivot
        g = random_graph(rng, num_nodes=40, num_events=600)
        for _ in range(300):
            v = int(rng.integers(0, g.num_nodes))
            t = float(rng.random() * 110)
            _, ts, _ = adjacency(g, v)
            assert pivot(g, v, t) == int((ts < t).sum())


class TestFindRecent:
    def test_definition(self):
        from paper_2402_05396_b200 import NeighborQuery, find_recent
        nb = find_recent(chain_graph([1.0, 5.0, 9.0, 12.0]), NeighborQuery(0, 10.0, 2))
        np.testing.assert_array_equal(nb.ts, [9.0, 5.0])

    def test_no_valid_neighbors(self):
        from paper_2402_05396_b200 import NeighborQuery, find_recent
        assert len(find_recent(chain_graph([1.0, 5.0]), NeighborQuery(0, 1.0, 3))) == 0

    def test_matches_sort_and_take_oracle(self, rng):
        from paper_2402_05396_b200 import NeighborQuery, find_recent
        g = random_graph(rng, num_nodes=25, num_events=500)
        for _ in range(150):
            q = NeighborQuery(int(rng.integers(0, 25)), float(rng.random() * 110), int(rng.integers(1, 8)))
            nb = find_recent(g, q)
            _, ts, eids = adjacency(g, q.v)
            valid = np.nonzero(ts < q.t)[0]
            np.testing.assert_array_equal(nb.eids, eids[valid[-q.m:][::-1]])


class TestFindUniform:
    def test_exhaustion_returns_all(self):
        from paper_2402_05396_b200 import NeighborQuery, find_uniform
        g = chain_graph([1.0, 2.0, 3.0])
        for seed in range(5):
            assert sorted(find_uniform(g, NeighborQuery(0, 10.0, 3), seed=seed).nodes) == [1, 2, 3]

    def test_empty_window(self):
        from paper_2402_05396_b200 import NeighborQuery, find_uniform
        assert len(find_uniform(chain_graph([5.0]), NeighborQuery(0, 1.0, 4), seed=0)) == 0

    def test_results_sorted_ts_descending(self, rng):
        from paper_2402_05396_b200 import NeighborQuery, find_uniform
        g = random_graph(rng, num_nodes=20, num_events=400)
        for seed in range(50):
            nb = find_uniform(g, NeighborQuery(int(rng.integers(0, 20)), 90.0, 5), seed=seed)
            assert (np.diff(nb.ts) <= 0).all()

    @pytest.mark.parametrize("p,m", [(20, 10), (9, 6), (12, 11)])
    def test_marginal_inclusion_frequency(self, p, m):
        from paper_2402_05396_b200 import batch_find_arrays
        g = chain_graph(list(np.arange(1.0, p + 1.0)))
        trials = 20_000
        idx, cnt = batch_find_arrays(g, np.zeros(trials, dtype=np.int64), np.full(trials, float(p + 1)), m,
                                     policy="uniform", seed=777)
        assert (cnt == m).all()
        counts = np.bincount(idx[:, :m].ravel(), minlength=p).astype(float)
        expected = trials * m / p
        chi2 = ((counts - expected) ** 2 / expected).sum()
        assert chi2 < stats.chi2.ppf(1 - 1e-3, df=p - 1)

    def test_no_duplicates_fuzz(self, rng):
        from paper_2402_05396_b200 import batch_find_arrays
        g = random_graph(rng, num_nodes=15, num_events=300)
        qv = rng.integers(0, 15, 2000).astype(np.int64)
        qt = rng.random(2000) * 110
        for m in (3, 7, 15):
            idx, cnt = batch_find_arrays(g, qv, qt, m, policy="uniform", seed=5)
            for i in range(2000):
                assert len(set(idx[i, :cnt[i]].tolist())) == cnt[i]

    def test_temporal_validity_fuzz(self, rng):
        from paper_2402_05396_b200 import batch_find_arrays
        g = random_graph(rng, num_nodes=15, num_events=300)
        qv = rng.integers(0, 15, 5000).astype(np.int64)
        qt = rng.random(5000) * 110
        idx, cnt = batch_find_arrays(g, qv, qt, 6, policy="uniform", seed=6)
        tts = _np(g.tcsr_ts)
        for i in range(5000):
            assert (tts[idx[i, :cnt[i]]] < qt[i]).all()


class TestBatchFind:
    def test_batch_of_one_matches_single(self, rng):
        from paper_2402_05396_b200 import NeighborQuery, batch_find, find_uniform
        g = random_graph(rng, num_nodes=20, num_events=300)
        q = NeighborQuery(3, 80.0, 5)
        np.testing.assert_array_equal(find_uniform(g, q, seed=42).eids,
                                      batch_find(g, [q], policy="uniform", seed=42)[0].eids)

    def test_worker_counts_bit_identical(self, rng):
        from paper_2402_05396_b200 import batch_find_arrays
        g = random_graph(rng, num_nodes=30, num_events=500)
        qv = rng.integers(0, 30, 500).astype(np.int64)
        qt = rng.random(500) * 110
        i1, c1 = batch_find_arrays(g, qv, qt, 8, policy="uniform", seed=9, workers=1)
        i8, c8 = batch_find_arrays(g, qv, qt, 8, policy="uniform", seed=9, workers=8)
        assert np.array_equal(i1, i8) and np.array_equal(c1, c8)

    def test_matches_sequential_scan(self, rng):
        """naive_scan_find (finder.py): the m most recent entries with ts < t."""
        from paper_2402_05396_b200 import NeighborQuery, batch_find
        g = random_graph(rng, num_nodes=30, num_events=500)
        queries = [NeighborQuery(int(rng.integers(0, 30)), float(rng.random() * 110), 5) for _ in range(300)]
        for q, nb in zip(queries, batch_find(g, queries, policy="recent", seed=1)):
            _, ts, eids = adjacency(g, q.v)
            sel = [e for t_, e in zip(ts[::-1], eids[::-1]) if t_ < q.t][:q.m]
            np.testing.assert_array_equal(nb.eids, sel)

    def test_uniform_set_matches_naive_window(self, rng):
        from paper_2402_05396_b200 import NeighborQuery, batch_find
        g = random_graph(rng, num_nodes=20, num_events=300)
        queries = [NeighborQuery(int(rng.integers(0, 20)), float(rng.random() * 110), 4) for _ in range(200)]
        for q, nb in zip(queries, batch_find(g, queries, policy="uniform", seed=3)):
            _, ts, eids = adjacency(g, q.v)
            window = set(eids[ts < q.t].tolist())
            assert set(nb.eids.tolist()) <= window and len(nb) == min(q.m, len(window))

    def test_mixed_budgets_rejected(self, rng):
        from paper_2402_05396_b200 import NeighborQuery, batch_find
        with pytest.raises(ValueError):
            batch_find(random_graph(rng), [NeighborQuery(0, 1.0, 2), NeighborQuery(0, 1.0, 3)])

    def test_same_seed_same_results_across_calls(self, rng):
        from paper_2402_05396_b200 import batch_find_arrays
        g = random_graph(rng, num_nodes=20, num_events=300)
        qv = rng.integers(0, 20, 100).astype(np.int64)
        qt = rng.random(100) * 110
        a = batch_find_arrays(g, qv, qt, 5, policy="uniform", seed=11)
        b = batch_find_arrays(g, qv, qt, 5, policy="uniform", seed=11)
        c = batch_find_arrays(g, qv, qt, 5, policy="uniform", seed=12)
        assert np.array_equal(a[0], b[0]) and not np.array_equal(a[0], c[0])


# ---------------------------------------------------------------- cache (test_cache.py)
class TestCacheLookup:
    def test_empty_resident_all_misses(self):
        from paper_2402_05396_b200 import lookup, make_cache
        state = make_cache(10, k=3)
        _, hits = lookup(state, [0, 1, 2])
        assert not hits.any() and state.epoch_stats[-1].misses == 3

    def test_repeat_request_counts_twice(self):
        from paper_2402_05396_b200 import lookup, make_cache
        state = make_cache(10, k=3)
        lookup(state, [4, 4])
        assert int(state.counters[4]) == 2

    def test_conservation_on_random_traces(self, rng):
        from paper_2402_05396_b200 import lookup, make_cache
        state = make_cache(50, k=5)
        total = 0
        for _ in range(20):
            eids = rng.integers(0, 50, rng.integers(1, 40))
            lookup(state, eids)
            total += eids.size
        st = state.epoch_stats[-1]
        assert st.hits + st.misses == total and int(state.counters.sum()) == total

    def test_unknown_eid_rejected(self):
        from paper_2402_05396_b200 import lookup, make_cache
        with pytest.raises(IndexError):
            lookup(make_cache(10, k=2), [10])

    def test_features_served_from_both_tiers(self, rng):
        from paper_2402_05396_b200 import lookup, make_cache
        feats = rng.normal(size=(10, 4)).astype(np.float32)
        state = make_cache(10, k=2, features=feats)
        state.slot_of[3] = 0  # resident (the reference sets state.resident[3] = True)
        got, hits = lookup(state, [3, 7])
        np.testing.assert_array_equal(got[:, :4], feats[[3, 7]])
        assert hits.tolist() == [True, False]


class TestCacheReplacement:
    def test_topk_definition(self):
        from paper_2402_05396_b200 import lookup, make_cache, maybe_replace
        state = make_cache(10, k=2, epsilon=1)
        lookup(state, [1] * 5 + [2] * 3 + [3])
        assert maybe_replace(state)
        assert set(np.nonzero(_np(state.resident))[0]) == {1, 2}

    def test_no_replacement_when_overlap_sufficient(self):
        from paper_2402_05396_b200 import lookup, make_cache, maybe_replace
        state = make_cache(10, k=2, epsilon=2)
        lookup(state, [1, 1, 2])
        maybe_replace(state)
        lookup(state, [1, 1, 2])
        assert maybe_replace(state) is False

    def test_counters_reset_either_way(self):
        from paper_2402_05396_b200 import lookup, make_cache, maybe_replace
        state = make_cache(10, k=2, epsilon=1)
        lookup(state, [1, 2, 3])
        maybe_replace(state)
        assert (_np(state.counters) == 0).all()

    def test_tie_at_kth_slot_lower_eid_wins(self):
        from paper_2402_05396_b200 import lookup, make_cache, maybe_replace
        for _ in range(3):
            state = make_cache(10, k=2, epsilon=2)
            lookup(state, [5, 7, 7, 9, 3])
            maybe_replace(state)
            assert tuple(np.nonzero(_np(state.resident))[0]) == (3, 7)

    def test_residency_bound_held(self, rng):
        from paper_2402_05396_b200 import lookup, make_cache, maybe_replace
        state = make_cache(30, k=4)
        for _ in range(15):
            lookup(state, rng.integers(0, 30, 25))
            maybe_replace(state)
            assert state.resident_count <= 4


class TestCacheOracle:
    def test_budget_covers_everything(self):
        from paper_2402_05396_b200 import oracle_cache
        counts = np.zeros((1, 10), dtype=int)
        counts[0, [1, 5]] = 3
        assert oracle_cache(counts, k=5) == [1.0]

    def test_zero_budget(self):
        from paper_2402_05396_b200 import oracle_cache
        assert oracle_cache(np.ones((2, 6), dtype=int), k=0) == [0.0, 0.0]

    def test_stationary_trace_matches_from_epoch_two(self, rng):
        from paper_2402_05396_b200 import make_cache, oracle_cache, run_trace
        epoch_eids = rng.integers(0, 40, 500)
        trace = [epoch_eids] * 4
        counts = np.stack([np.bincount(e, minlength=40) for e in trace])
        rates = run_trace(make_cache(40, k=6), trace)
        np.testing.assert_allclose(rates[1:], oracle_cache(counts, 6)[1:])

    def test_oracle_dominates_every_epoch(self, rng):
        from paper_2402_05396_b200 import make_cache, oracle_cache, run_trace
        for _ in range(10):
            trace = [rng.integers(0, 30, rng.integers(10, 200)) for _ in range(5)]
            counts = np.stack([np.bincount(e, minlength=30) for e in trace])
            rates = run_trace(make_cache(30, k=5), trace)
            for r, o in zip(rates, oracle_cache(counts, 5)):
                assert o >= r - 1e-12

    def test_oracle_monotone_in_budget(self, rng):
        from paper_2402_05396_b200 import oracle_cache
        counts = np.bincount(rng.integers(0, 50, 800), minlength=50)[None, :]
        rates = [oracle_cache(counts, k)[0] for k in range(0, 51, 5)]
        assert all(b >= a for a, b in zip(rates, rates[1:]))


class TestCacheReport:
    def test_zero_denominator_flagged(self):
        from paper_2402_05396_b200 import cache_report, make_cache, maybe_replace
        state = make_cache(10, k=2)
        maybe_replace(state)
        rep = cache_report(state)
        assert rep["epochs"][0]["zero_denominator"] and rep["epochs"][0]["hit_rate"] is None

    def test_json_roundtrip(self, rng):
        from paper_2402_05396_b200 import cache_report, make_cache, run_trace
        state = make_cache(20, k=3)
        run_trace(state, [rng.integers(0, 20, 50) for _ in range(3)])
        rep = cache_report(state, oracle_rates=[0.5, 0.6, 0.7])
        assert json.loads(json.dumps(rep)) == rep

    def test_fraction_budget_and_epsilon(self):
        from paper_2402_05396_b200 import make_cache
        state = make_cache(100, k=0.1)
        assert state.k == 10 and state.epsilon == 9


# ---------------------------------------------------------------- sampler (test_sampler.py)
DECODERS = ("linear", "gat", "gatv2", "trans")


def build_policy_inputs(rng, d=3, m=4, B=2, d_v=2, d_e=2, seed=0, decoder="linear"):
    """The reference's build_policy_inputs: a balanced EncoderConfig, a
    fresh sampler store (ParamStore-identical init), random candidates."""
    from paper_2402_05396_b200 import EncoderConfig, encode_neighborhood_batch, encode_target_batch
    from paper_2402_05396_b200.params import sampler_params
    ecfg = EncoderConfig.balanced(d, m)
    store = sampler_params(seed, d, m, d_v, d_e, decoder)
    ids = rng.integers(0, 6, (B, m))
    dts = rng.random((B, m)) * 3
    mask = np.ones((B, m), dtype=bool)
    node_rows = rng.normal(size=(B, m, d_v)).astype(np.float32) if d_v else None
    edge_rows = rng.normal(size=(B, m, d_e)).astype(np.float32) if d_e else None
    z_raw = encode_neighborhood_batch(ids, dts, mask, node_rows, edge_rows, ecfg, store)
    tgt_rows = rng.normal(size=(B, d_v)).astype(np.float32) if d_v else None
    z_target = encode_target_batch(np.zeros(B, dtype=np.int64), tgt_rows, ecfg, store)
    return ecfg, store, z_raw, z_target, mask, (d_v, d_e), (ids, dts, node_rows, edge_rows, tgt_rows)


class TestMixerTransform:
    def test_zero_input_zero_weights_gives_zero(self, rng):
        import torch
        from paper_2402_05396_b200 import mixer_transform
        _, store, z_raw, _, mask, _, _ = build_policy_inputs(rng)
        for name in store:
            if name.startswith("sampler/mixer") and ("ln" not in name or "beta" in name):
                store[name] = np.zeros_like(store[name])
        out = mixer_transform(torch.zeros(z_raw.shape, dtype=torch.float64, device="cuda"), mask, store)
        assert not _np(out).any()

    def test_output_shape_and_masked_rows(self, rng):
        from paper_2402_05396_b200 import mixer_transform
        _, store, z_raw, _, mask, _, _ = build_policy_inputs(rng, B=3)
        mask[1, 2:] = False
        out = mixer_transform(z_raw, mask, store)
        assert tuple(out.shape) == tuple(z_raw.shape)
        assert not _np(out)[~mask].any()


class TestDecoders:
    @pytest.mark.parametrize("kind", DECODERS)
    def test_probability_validity(self, kind, rng):
        from paper_2402_05396_b200 import SamplerConfig, decode_policy, mixer_transform
        ecfg, store, z_raw, z_target, mask, (d_v, d_e), _ = build_policy_inputs(rng, B=3, decoder=kind)
        mask[0, 1] = False
        mask[2, 2:] = False
        scfg = SamplerConfig(decoder=kind, n=2, m=4)
        pol = decode_policy(z_raw, mixer_transform(z_raw, mask, store), z_target, mask, scfg, ecfg, store, d_v, d_e)
        q = _np(pol.q)
        assert (q >= 0).all()
        np.testing.assert_allclose(q.sum(axis=1), 1.0)
        assert not q[~mask].any()
        assert np.isfinite(_np(pol.log_q)[mask]).all()

    def test_linear_zero_weights_uniform(self, rng):
        from paper_2402_05396_b200 import SamplerConfig, decode_policy, mixer_transform
        ecfg, store, z_raw, z_target, mask, (d_v, d_e), _ = build_policy_inputs(rng)
        store["sampler/w_linear"] = np.zeros_like(store["sampler/w_linear"])
        scfg = SamplerConfig(decoder="linear", n=2, m=4)
        pol = decode_policy(z_raw, mixer_transform(z_raw, mask, store), z_target, mask, scfg, ecfg, store, d_v, d_e)
        np.testing.assert_allclose(_np(pol.q), 0.25)

    @pytest.mark.parametrize("kind", DECODERS)
    def test_single_valid_slot(self, kind, rng):
        from paper_2402_05396_b200 import SamplerConfig, decode_policy, mixer_transform
        ecfg, store, z_raw, z_target, mask, (d_v, d_e), _ = build_policy_inputs(rng, decoder=kind)
        mask[:] = False
        mask[:, 1] = True
        scfg = SamplerConfig(decoder=kind, n=1, m=4)
        pol = decode_policy(z_raw, mixer_transform(z_raw, mask, store), z_target, mask, scfg, ecfg, store, d_v, d_e)
        np.testing.assert_allclose(_np(pol.q)[:, 1], 1.0)

    def test_trans_rescaling_invariance(self, rng):
        from paper_2402_05396_b200 import SamplerConfig, decode_policy, mixer_transform
        ecfg, store, z_raw, z_target, mask, (d_v, d_e), _ = build_policy_inputs(rng, decoder="trans")
        scfg = SamplerConfig(decoder="trans", n=2, m=4)
        zm = mixer_transform(z_raw, mask, store)
        q1 = _np(decode_policy(z_raw, zm, z_target, mask, scfg, ecfg, store, d_v, d_e).q)
        store["sampler/W_trans_target"] = store["sampler/W_trans_target"] * 2.0
        store["sampler/W_trans_nbr"] = store["sampler/W_trans_nbr"] * 0.5
        q2 = _np(decode_policy(z_raw, zm, z_target, mask, scfg, ecfg, store, d_v, d_e).q)
        np.testing.assert_allclose(q1, q2, atol=1e-12)

    def test_unknown_decoder_rejected(self):
        from paper_2402_05396_b200 import ConfigError, SamplerConfig
        with pytest.raises(ConfigError):
            SamplerConfig(decoder="mlp", n=2, m=4)

    @pytest.mark.parametrize("kind", DECODERS)
    def test_decoder_gradients(self, kind, rng):
        """d/dtheta sum(w * log_q * mask) through decoder, mixer and encoders:
        the device backward against central differences of the device f64
        forward (the reference checks its autodiff the same way, rtol 2e-4)."""
        import torch
        from paper_2402_05396_b200.params import ScoringModel
        from paper_2402_05396_b200.scoring import SamplerGrad, score_policy
        ecfg, store, _, _, mask, (d_v, d_e), (ids, dts, nr, er, tr) = build_policy_inputs(
            rng, B=1, seed=7 + DECODERS.index(kind), decoder=kind)
        model = ScoringModel(store, kind, ecfg.d_feat, ecfg.m, d_v, d_e, ecfg.alpha, ecfg.beta, precision="float64")
        dev = lambda a, dt: torch.as_tensor(a).to("cuda", dt)  # noqa: E731
        args = (dev(ids, torch.int64), dev(dts, torch.float64), dev(mask, torch.bool), dev(nr, torch.float32),
                dev(er, torch.float32), dev(tr, torch.float32))
        w = rng.normal(size=(1, 4)) * mask

        def loss():
            _, lq = score_policy(model, *args)
            return float((_np(lq) * w).sum())

        q, _ = score_policy(model, *args)
        g = w * mask
        dl = g - _np(q) * g.sum(axis=1, keepdims=True)
        sg = SamplerGrad(model)
        sg.backward(args[0], args[1], args[2], torch.as_tensor(dl).cuda(), node_rows=args[3], edge_rows=args[4],
                    tgt_rows=args[5])
        eps = 1e-6
        for name, p in model.named_params().items():
            got = _np(sg.grads[name])
            num = np.zeros(p.numel())
            for i in range(p.numel()):
                old = float(p[i])
                p[i] = old + eps
                lp = loss()
                p[i] = old - eps
                lm = loss()
                p[i] = old
                num[i] = (lp - lm) / (2 * eps)
            np.testing.assert_allclose(got, num, rtol=2e-4, atol=1e-7, err_msg=f"{kind} {name}")


def logits_policy(theta, mask=None):
    """Policy parameterised by raw logits: q / log q by the reference's masked
    (log-)softmax definition (autodiff.py:429-464), computed on the host."""
    from paper_2402_05396_b200 import PolicyOutput
    B, m = theta.shape
    mask = np.ones((B, m), dtype=bool) if mask is None else mask
    x = np.where(mask, theta, -np.inf)
    mx = np.max(x, axis=1, keepdims=True)
    e = np.where(mask, np.exp(theta - mx), 0.0)
    z = e.sum(axis=1, keepdims=True)
    return PolicyOutput(q=e / z, log_q=np.where(mask, theta - mx - np.log(z), -1e30), mask=mask)


class TestSampling:
    def test_exhaustion_returns_all_slots(self, rng):
        from paper_2402_05396_b200 import sample_without_replacement
        pol = sample_without_replacement(logits_policy(np.zeros((1, 4))), 4, rng)
        assert sorted(pol.selected[0].tolist()) == [0, 1, 2, 3]

    def test_degenerate_distribution(self, rng):
        from paper_2402_05396_b200 import sample_without_replacement
        pol = logits_policy(np.array([[50.0, -50.0, -50.0, -50.0]]))
        for _ in range(20):
            assert sample_without_replacement(pol, 1, rng).selected[0, 0] == 0

    def test_short_neighborhood_returns_valid_only(self, rng):
        from paper_2402_05396_b200 import sample_without_replacement
        pol = sample_without_replacement(logits_policy(np.zeros((1, 4)), np.array([[True, True, False, False]])), 3,
                                         rng)
        assert sorted(pol.selected[0, :2].tolist()) == [0, 1]
        assert pol.selected[0, 2] == -1 and pol.selected_mask[0].tolist() == [True, True, False]

    def test_empirical_frequencies_match_q(self):
        from paper_2402_05396_b200 import sample_without_replacement
        probs = np.array([0.7, 0.2, 0.1])
        pol = logits_policy(np.log(probs)[None, :])
        rng = np.random.default_rng(99)
        trials = 20_000
        counts = np.zeros(3)
        for _ in range(trials):
            counts[sample_without_replacement(pol, 1, rng).selected[0, 0]] += 1
        se = np.sqrt(probs * (1 - probs) / trials)
        assert (np.abs(counts / trials - probs) <= 3 * se + 1e-9).all()

    def test_selected_log_q_matches_original_q(self, rng):
        from paper_2402_05396_b200 import sample_without_replacement
        pol = sample_without_replacement(logits_policy(rng.normal(size=(2, 4))), 2, rng)
        for b in range(2):
            for i in range(2):
                np.testing.assert_allclose(pol.selected_log_q[b, i], pol.log_q[b, pol.selected[b, i]])

    def test_selection_sorted_most_recent_first(self, rng):
        from paper_2402_05396_b200 import sample_without_replacement
        sel = sample_without_replacement(logits_policy(np.zeros((4, 6))), 3, rng).selected
        assert (np.diff(sel, axis=1) > 0).all()


# ---------------------------------------------------------------- encoders (test_encoders.py)
class TestEncoders:
    def test_masked_rows_exactly_zero_and_width(self, rng):
        from paper_2402_05396_b200 import EncoderConfig, encode_neighborhood_batch
        from paper_2402_05396_b200.encoders import encoded_width
        from paper_2402_05396_b200.params import sampler_params
        ecfg = EncoderConfig.balanced(5, 6)
        store = sampler_params(3, 5, 6, 4, 3, "linear")
        mask = rng.random((7, 6)) < 0.6
        z = _np(encode_neighborhood_batch(rng.integers(0, 4, (7, 6)), rng.random((7, 6)) * 50, mask,
                                          rng.normal(size=(7, 6, 4)), rng.normal(size=(7, 6, 3)), ecfg, store))
        assert z.shape == (7, 6, encoded_width(ecfg, 4, 3))
        assert not z[~mask].any()

    def test_absent_feature_kinds_consume_no_columns(self, rng):
        from paper_2402_05396_b200 import EncoderConfig, encode_neighborhood_batch, encode_target_batch
        from paper_2402_05396_b200.params import sampler_params
        ecfg = EncoderConfig.balanced(4, 3)
        store = sampler_params(1, 4, 3, 0, 0, "linear")
        z = encode_neighborhood_batch(np.zeros((2, 3), dtype=np.int64), np.zeros((2, 3)), np.ones((2, 3), bool), None,
                                      None, ecfg, store)
        assert tuple(z.shape) == (2, 3, 4 + 4 + 3)
        zt = _np(encode_target_batch(np.zeros(2, dtype=np.int64), None, ecfg, store))
        assert zt.shape == (2, 8)
        np.testing.assert_allclose(zt[:, :4], 1.0)  # cos(0 * omega)

    def test_identity_and_frequency_blocks(self):
        from paper_2402_05396_b200 import EncoderConfig, encode_neighborhood_batch
        from paper_2402_05396_b200.params import freq_table, sampler_params
        ecfg = EncoderConfig.balanced(4, 4)
        store = sampler_params(0, 4, 4, 0, 0, "linear")
        ids = np.array([[7, 7, 2, 7]])
        mask = np.array([[True, True, True, False]])
        z = _np(encode_neighborhood_batch(ids, np.zeros((1, 4)), mask, None, None, ecfg, store))[0]
        ie = z[:, 8:]
        np.testing.assert_array_equal(ie[:3, :3], [[1, 1, 0], [1, 1, 0], [0, 0, 1]])
        fe = freq_table(4, 4)
        np.testing.assert_allclose(z[0, 4:8], fe[2])
        np.testing.assert_allclose(z[2, 4:8], fe[1])

    def test_balanced_only(self):
        from paper_2402_05396_b200 import ConfigError, EncoderConfig, encode_neighborhood_batch
        with pytest.raises(ConfigError):
            encode_neighborhood_batch(np.zeros((1, 2), dtype=np.int64), np.zeros((1, 2)), np.ones((1, 2), bool), None,
                                      None, EncoderConfig(d_time=3, d_freq=4, d_feat=3, m=2), {})



# ---------------------------------------------------------------- staged forward vs golden
@pytest.mark.parametrize("tag", [f"s{i}" for i in range(8)])
def test_stages_match_reference_scoring(tag):
    """encode_neighborhood_batch -> mixer_transform -> encode_target_batch ->
    decode_policy through the drop-ins reproduce the reference's z_raw /
    z_mixed / z_target (where stored) and q / log q (golden scoring.npz, f64,
    <= 1e-11 relative)."""
    from conftest import load_golden
    from paper_2402_05396_b200 import (EncoderConfig, SamplerConfig, decode_policy, encode_neighborhood_batch,
                                       encode_target_batch, mixer_transform)
    from paper_2402_05396_b200.params import sampler_params
    z = load_golden("scoring")
    d_v, d_e, enc, m, B, store_seed = (int(x) for x in z[f"{tag}/meta"])
    dec = str(z[f"{tag}/decoder"])
    alpha, beta, _ = (float(x) for x in z[f"{tag}/ab"])
    store = sampler_params(store_seed, enc, m, d_v, d_e, dec)
    ecfg = EncoderConfig.balanced(enc, m, alpha=alpha, beta=beta)
    scfg = SamplerConfig(decoder=dec, n=min(3, m), m=m)
    mask = z[f"{tag}/mask"]
    nr = z[f"{tag}/node_rows"] if d_v else None
    er = z[f"{tag}/edge_rows"] if d_e else None
    tr = z[f"{tag}/tgt_rows"] if d_v else None
    zr = encode_neighborhood_batch(z[f"{tag}/ids"], z[f"{tag}/dts"], mask, nr, er, ecfg, store)
    zm = mixer_transform(zr, mask, store)
    zt = encode_target_batch(np.arange(B), tr, ecfg, store)
    pol = decode_policy(zr, zm, zt, mask, scfg, ecfg, store, d_v, d_e)
    if f"{tag}/z_raw" in z.files:
        np.testing.assert_allclose(_np(zr), z[f"{tag}/z_raw"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(_np(zm), z[f"{tag}/z_mixed"], rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(_np(zt), z[f"{tag}/z_target"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(_np(pol.q), z[f"{tag}/q"], rtol=1e-11, atol=1e-14)
    lq, rlq = _np(pol.log_q), z[f"{tag}/log_q"]
    np.testing.assert_allclose(lq[mask], rlq[mask], rtol=1e-11, atol=1e-12)
