"""K9 (select.cu) against the reference's importance-weighted selection
(selector.py:46-61) -- golden vectors of the real reference plus the CPU
oracle at larger sizes.  Selection is bit-exact (same PCG64 stream, numpy's
pairwise total and sequential cumsum reproduced); update_scores differs from
numpy only through exp() rounding (<= 2 ulp, checked)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _np(x):
    return x.detach().cpu().numpy()


def _ulps(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64).view(np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64).view(np.int64)
    return np.abs(a - b)


@pytest.mark.parametrize("ci", range(9))
def test_device_select_batch_matches_reference(ci):
    import torch
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    z = load_golden("selector")
    n, b, seed, base = (int(x) for x in z[f"c{ci}/meta"])
    host = osel.case_scores(str(z[f"c{ci}/kind"]), n, seed)
    for it in range(3):
        p = f"c{ci}/it{it}"
        sc = dsel.as_scores(host, 0.1, base_eid=base)
        rng = osel.pcg_generator(z[p + "/pcg"])
        eids = dsel.select_batch(sc, b, rng)
        np.testing.assert_array_equal(_np(eids), z[p + "/eids"], err_msg=f"case {ci} it {it}")
        # the caller's generator advanced exactly like numpy's choice()
        ref_rng = osel.pcg_generator(z[p + "/pcg"])
        osel.select_batch(host.copy(), b, ref_rng)
        assert rng.bit_generator.state["state"] == ref_rng.bit_generator.state["state"]
        # Eq. 10 update on the device vs numpy (exp rounding only)
        dsel.update_scores(sc, eids, torch.as_tensor(z[p + "/logits"]).cuda())
        osel.update_scores(host, z[p + "/eids"], z[p + "/logits"], 0.1, base_eid=base)
        assert _ulps(_np(sc.scores), host).max() <= 2
        # continue the chain from the reference's own scores
        if p + "/scores_after" in z:
            assert host.tobytes() == z[p + "/scores_after"].tobytes()


@pytest.mark.parametrize("kind,n,b", [("short", 20_000_000, 600), ("random", 8_000_000, 2000),
                                      ("skewed", 3_000_001, 600), ("init", 12_000_000, 600)])
def test_device_select_batch_large_vs_oracle(kind, n, b):
    """Millions of rows: thousands of fast chunks, binade crossings and (for
    integer scores) rounding ties, bit-exact against numpy's choice."""
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    host = osel.case_scores(kind, n, 99)
    for it in range(2):
        words = np.array([it, 12345 + it, 0, 2 * it + 1], dtype=np.uint64)
        exp = osel.select_batch(host, b, osel.pcg_generator(words), base_eid=7)
        got = dsel.select_batch(dsel.as_scores(host, 0.1, base_eid=7), b, osel.pcg_generator(words))
        np.testing.assert_array_equal(_np(got), exp)


def test_device_select_batch_multi_round_and_full():
    """b close to n forces many choice() rounds; b == n returns every row."""
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    r = np.random.default_rng(4)
    for n, b in ((40, 39), (500, 480), (3000, 3000), (70, 1)):
        host = r.random(n) ** 4 + 1e-3
        for s in range(3):
            words = np.array([0, 77 + s, 0, 11], dtype=np.uint64)
            exp = osel.select_batch(host, b, osel.pcg_generator(words))
            got = dsel.select_batch(dsel.as_scores(host, 0.1), b, osel.pcg_generator(words))
            np.testing.assert_array_equal(_np(got), exp)


def test_device_select_batch_errors():
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    g = lambda: osel.pcg_generator(np.array([0, 1, 0, 3], dtype=np.uint64))  # noqa: E731
    with pytest.raises(ValueError, match="exceeds"):
        dsel.select_batch(dsel.as_scores(np.ones(5), 0.1), 6, g())
    with pytest.raises(ValueError, match="non-zero"):
        dsel.select_batch(dsel.as_scores(np.array([1.0, 0.0, 0.0, 2.0]), 0.1), 3, g())
    with pytest.raises(ValueError, match="NaN"):
        dsel.select_batch(dsel.as_scores(np.zeros(4), 0.1), 2, g())
    with pytest.raises(ValueError, match="non-negative"):
        dsel.select_batch(dsel.as_scores(np.array([1.0, -1.0, 2.0]), 0.1), 1, g())
    sc = dsel.init_scores(10, gamma=0.2, base_eid=100)
    assert np.all(_np(sc.scores) == 0.7)
    with pytest.raises(IndexError):
        dsel.update_scores(sc, [100, 110], [0.0, 1.0])
    with pytest.raises(dsel.IndexError_):
        dsel.update_scores(sc, [99], [0.0])
    dsel.update_scores(sc, [100, 100, 105], [5.0, -3.0, 0.0])  # duplicate eid: the last write wins
    got = _np(sc.scores)
    assert _ulps(got[[0, 5]], osel.sigmoid([-3.0, 0.0]) + 0.2).max() <= 2


def test_device_generator_select_roots_matches_oracle():
    """MiniBatchGenerator(adaptive_minibatch) roots = the Trainer's
    (training.py:364-382): select_batch on S_BATCH, positives gathered,
    negatives from S_NEG; then Eq. 10 updates steer the next selection."""
    import torch
    from oracle import selector as osel
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.seeds import S_BATCH, S_NEG, substream
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["E"].scaled(0.0002)
    og = oshapes.make_graph(spec, seed=8)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = PathConfig(aggregator="tgat", finder_policy="recent", adaptive_neighbor=False, n=10, batch_size=200,
                     adaptive_minibatch=True, gamma=0.1)
    gen = MiniBatchGenerator(g, cfg, seed=3)
    lo, hi = gen.train_lo, gen.train_hi
    host = np.full(hi - lo, 0.6)
    pool = gen.dst_pool()
    for it in range(4):
        nodes, times, eids = gen.select_roots(it)
        exp = osel.select_batch(host, 200, substream(3, S_BATCH, it), base_eid=lo)
        np.testing.assert_array_equal(_np(eids), exp)
        negs = pool[substream(3, S_NEG, it).integers(0, pool.size, size=200)]
        np.testing.assert_array_equal(_np(nodes), np.concatenate([og.src[exp], og.dst[exp], negs]))
        assert _np(times).tobytes() == np.concatenate([og.ts[exp]] * 3).tobytes()
        logits = np.random.default_rng(it).normal(size=200) * 3
        gen.update_scores(eids, torch.as_tensor(logits).cuda())
        osel.update_scores(host, exp, logits, 0.1, base_eid=lo)
        host = _np(gen.scores.scores).copy()  # follow the device scores (exp may differ by an ulp)
        recs = gen.generate(nodes, times, it)
        assert int(recs[-1]["sel_mask"].sum()) > 0


def test_device_select_update_chain_bit_exact_with_host_logits():
    """Several select -> Eq. 10 rounds with HOST logits (the reference passes
    pos_logits.data, numpy): the scores stay bit-identical to the oracle's, so
    every later selection is bit-exact too (no resync from the device)."""
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    n, b, base = 300_000, 600, 11
    host = np.full(n, 0.6)
    sc = dsel.as_scores(host.copy(), 0.1, base_eid=base)
    for it in range(6):
        words = np.array([it, 99 + it, 0, 5], dtype=np.uint64)
        exp = osel.select_batch(host, b, osel.pcg_generator(words), base_eid=base)
        got = _np(dsel.select_batch(sc, b, osel.pcg_generator(words)))
        np.testing.assert_array_equal(got, exp, err_msg=f"round {it}")
        logits = np.random.default_rng(it).normal(size=b) * 4
        dsel.update_scores(sc, got, logits)
        osel.update_scores(host, exp, logits, 0.1, base_eid=base)
        assert _np(sc.scores).tobytes() == host.tobytes(), f"round {it}: scores differ"


@pytest.mark.parametrize("b", [7, 600, 4096, 5000])
def test_device_update_scores_duplicates_last_writer(b):
    """numpy fancy assignment: a repeated eid keeps its LAST position's value
    (sorted single-CTA path up to 4096 positions, pairwise path above)."""
    import torch
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    r = np.random.default_rng(b)
    n = 3 * b
    eids = r.integers(0, max(2, b // 3), size=b) + 40
    logits = r.normal(size=b)
    for host_logits in (True, False):
        sc = dsel.as_scores(np.full(n, 0.6), 0.1, base_eid=40)
        ref = np.full(n, 0.6)
        dsel.update_scores(sc, eids, logits if host_logits else torch.as_tensor(logits).cuda())
        osel.update_scores(ref, eids, logits, 0.1, base_eid=40)
        got = _np(sc.scores)
        if host_logits:
            assert got.tobytes() == ref.tobytes()
        else:
            assert _ulps(got, ref).max() <= 2
