"""Parity of the round-2 device paths: the finder's coarse time index
(tg_tcsr_coarse) and the multi-segment K5 launch (tg_gather_rows_multi),
each against the plain path and the CPU oracle, bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _np(x):
    return x.detach().cpu().numpy()


def _tie_heavy_hubs(E=400_000, V=40, seed=5):
    """Few nodes (windows of ~20k entries) with integer timestamps repeated
    ~8 times each, so coarse-block boundaries fall inside runs of ties."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    ts = np.sort(np.floor(rng.random(E) * (E / 8))).astype(np.float64)
    return src, dst, ts


@pytest.mark.parametrize("shift", [1, 4, 6, 9])
def test_device_coarse_index_pivots_match_plain_search_and_oracle(shift):
    import torch
    from oracle import finder as ofinder
    from oracle import tcsr as otcsr
    from paper_2402_05396_b200 import batch_find_arrays, build_graph
    src, dst, ts = _tie_heavy_hubs()
    g = build_graph(src, dst, ts, num_nodes=40)
    og = otcsr.build_graph(src, dst, ts, num_nodes=40)
    rng = np.random.default_rng(1)
    qv = rng.integers(0, 40, 30000)
    # query times: existing timestamps (strict-< ties), midpoints, and out of range
    qt = np.concatenate([ts[rng.integers(0, ts.size, 10000)], ts[rng.integers(0, ts.size, 10000)] + 0.5,
                         rng.random(10000) * (ts[-1] + 10) - 5])
    g.coarse_shift = shift
    g._coarse = None
    res = {}
    for policy, m in (("recent", 10), ("uniform", 25)):
        i1, c1 = batch_find_arrays(g, qv, qt, m, policy=policy, seed=9)
        i2, c2 = ofinder.batch_find_arrays(og, qv, qt, m, policy=policy, seed=9)
        np.testing.assert_array_equal(i1, i2)
        np.testing.assert_array_equal(c1, c2)
        res[policy] = (i1, c1)
    # the same queries with the index switched off
    g.coarse_shift = 0
    for policy, m in (("recent", 10), ("uniform", 25)):
        i0, c0 = batch_find_arrays(g, qv, qt, m, policy=policy, seed=9)
        np.testing.assert_array_equal(i0, res[policy][0])
        np.testing.assert_array_equal(c0, res[policy][1])
    torch.cuda.synchronize()


def test_device_coarse_index_layout():
    """coarse_ts[coarse_off[v] + i] == adj_ts[offsets[v] + (i << s)]."""
    from paper_2402_05396_b200 import build_graph
    src, dst, ts = _tie_heavy_hubs(E=50_000, V=300)
    g = build_graph(src, dst, ts, num_nodes=300)
    g.c_graph()
    coff, cts = (_np(x) for x in g._coarse)
    off, adj = _np(g.tcsr_offsets), _np(g.tcsr_ts)
    s = g.coarse_shift
    for v in range(300):
        n = off[v + 1] - off[v]
        nb = (n + (1 << s) - 1) >> s
        assert coff[v + 1] - coff[v] == nb
        np.testing.assert_array_equal(cts[coff[v]:coff[v + 1]], adj[off[v]:off[v + 1]][::1 << s])


@pytest.mark.parametrize("ring", ["16x2", "16x3", "16x4", "16x6", "32x2", "32x3", "32x4", "32x6"])
@pytest.mark.parametrize("d", [186, 266])
@pytest.mark.parametrize("sizes", [(18000, 198000), (1, 2, 3, 4, 5, 6, 7), (0, 37, 0, 5)])
def test_device_gather4_tile_rings_match(sizes, d, ring, monkeypatch):
    """The gather4 K5 at every tile height / ring depth (TG_K5_G4_ROWS,
    TG_K5_G4_STAGES): the same rows as the per-segment gathers."""
    rows, stages = ring.split("x")
    monkeypatch.setenv("TG_K5_G4_ROWS", rows)
    monkeypatch.setenv("TG_K5_G4_STAGES", stages)
    test_device_gather_rows_multi_matches_per_segment(sizes, False, d, True, monkeypatch)


@pytest.mark.parametrize("sizes", [(18000, 198000), (0, 37, 0, 5), (1, 2, 3, 4, 5, 6, 7), (64000,)])
@pytest.mark.parametrize("hot", [False, True])
@pytest.mark.parametrize("d", [186, 266, 100])
@pytest.mark.parametrize("g4", [True, False])
def test_device_gather_rows_multi_matches_per_segment(sizes, hot, d, g4, monkeypatch):
    import torch
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200 import cache as dcache
    from paper_2402_05396_b200.graph import padded_rows, row_pitch
    # the gather4 path normally needs a DRAM-sized table: force it (or not) here
    monkeypatch.setenv("TG_K5_G4_MIN_MB", "0" if g4 else "1e12")
    rng = np.random.default_rng(len(sizes) + 10 * hot + d)
    E = 20000
    table = padded_rows((E,), d, "cuda")
    table.copy_(torch.as_tensor(rng.normal(size=(E, d)).astype(np.float32)).cuda())
    st = dcache.make_cache(E, 0.2, features=table, hot_tier=hot)
    dcache.lookup(st, torch.as_tensor(np.minimum(rng.zipf(1.3, 50000) - 1, E - 1)).cuda())
    dcache.maybe_replace(st)
    store = st.c_store() if hot else None
    if store is None:
        from paper_2402_05396_b200.graph import feat_store
        store = feat_store(table)
    pitch = row_pitch(d)
    segs, outs, refs = [], [], []
    for n in sizes:
        ids = torch.as_tensor(rng.integers(0, E, max(n, 1))[:n]).cuda()
        mask = torch.as_tensor(rng.random(n) < 0.8).cuda()
        out = torch.full((max(n, 1), pitch), float("nan"), device="cuda")
        ref = torch.full((max(n, 1), pitch), float("nan"), device="cuda")
        _lib.check(_lib.lib.tg_gather_rows(_lib.ptr(ids), _lib.ptr(mask), n, store, _lib.ptr(st.slot_of), 0,
                                           _lib.ptr(ref), pitch, _lib.stream_ptr()))
        segs.append(_lib.tg_gather_seg(_lib.ptr(ids), _lib.ptr(mask), n, _lib.ptr(out)))
        outs.append(out)
        refs.append((ref, ids, mask))
    arr = (_lib.tg_gather_seg * len(segs))(*segs)
    _lib.check(_lib.lib.tg_gather_rows_multi(arr, len(segs), store, _lib.ptr(st.slot_of), 0, pitch,
                                             _lib.stream_ptr()))
    torch.cuda.synchronize()
    for n, out, (ref, ids, mask) in zip(sizes, outs, refs):
        assert out[:n, :d].view(torch.int32).equal(ref[:n, :d].view(torch.int32))
        exp = torch.where(mask[:, None], table[ids][:, :d], torch.zeros((), device="cuda"))
        assert out[:n, :d].view(torch.int32).equal(exp.view(torch.int32))


def test_device_gather_rows_multi_validation():
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.graph import feat_store
    import torch
    table = torch.zeros((10, 4), device="cuda")
    seg = _lib.tg_gather_seg(None, None, -1, None)
    with pytest.raises(ValueError, match="negative row count"):
        _lib.check(_lib.lib.tg_gather_rows_multi(_lib.ctypes.byref(seg), 1, feat_store(table), None, 0, 4,
                                                 _lib.stream_ptr()))
    with pytest.raises(ValueError, match="mask_mode"):
        _lib.check(_lib.lib.tg_gather_rows_multi(_lib.ctypes.byref(seg), 1, feat_store(table), None, 3, 4,
                                                 _lib.stream_ptr()))


def test_device_generator_merged_gather_matches_per_layer():
    """generate() with every layer's rows in one K5 launch == per-layer launches."""
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["E"].scaled(0.0005)
    og = oshapes.make_graph(spec, seed=3)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = spec.path_config(batch_size=200)
    outs = []
    for merge in (True, False):
        gen = MiniBatchGenerator(g, cfg, seed=0)
        gen.merge_gathers = merge
        it = gen.iters_per_epoch // 3
        n, t = gen.roots_for_iteration(it)
        recs = gen.generate(torch.as_tensor(n).cuda(), torch.as_tensor(t).cuda(), it)
        torch.cuda.synchronize()
        outs.append([{k: _np(r[k]).copy() for k in ("sel_eids", "sel_mask", "edge_rows")} for r in recs] +
                    [_np(gen.cache.counters_i32).copy()])
    for a, b in zip(outs[0][:-1], outs[1][:-1]):
        for k in a:
            assert a[k].tobytes() == b[k].tobytes(), k
    np.testing.assert_array_equal(outs[0][-1], outs[1][-1])


@pytest.mark.parametrize("policy", ["recent", "uniform"])
def test_device_generate_batched_matches_generate(policy):
    """Several batches through one finder launch per layer + one K5 launch
    (generate_batched) == generate per batch, including the cache counts."""
    import torch
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["B"].scaled(0.05)
    og = oshapes.make_graph(spec, seed=4)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = PathConfig(aggregator="tgat", finder_policy=policy, adaptive_neighbor=False, n=10, batch_size=120)
    its = [3, 7, 11, 19, 23]
    res = []
    for batched in (False, True):
        gen = MiniBatchGenerator(g, cfg, seed=1)
        roots = [gen.roots_for_iteration(it) for it in its]
        dn = [(torch.as_tensor(n).cuda(), torch.as_tensor(t).cuda()) for n, t in roots]
        seeds = [torch.as_tensor([x - (1 << 64) if x >= (1 << 63) else x
                                  for x in (gen.seeds_for(it)[l] for l in range(gen.L, 0, -1))],
                                 dtype=torch.int64).cuda() for it in its]
        if batched:
            recs = gen.generate_batched([(n, t, sd, ("b", k)) for k, ((n, t), sd) in enumerate(zip(dn, seeds))])
        else:
            recs = []
            for (n, t), it in zip(dn, its):  # slot 0 reuses its buffers: copy each batch out
                rr = gen.generate(n, t, it, slot=0)
                recs.append([{k: v.clone() if hasattr(v, "clone") else v for k, v in r.items()} for r in rr])
        torch.cuda.synchronize()
        res.append(([[{k: _np(r[k]).copy() for k in ("sel_ids", "sel_eids", "sel_dts", "sel_mask", "edge_rows")}
                      for r in rr] for rr in recs], _np(gen.cache.counters_i32).copy(), _np(gen.cache.stats).copy()))
    (a, ca, sa), (b, cb, sb) = res
    for ra, rb in zip(a, b):
        for la, lb in zip(ra, rb):
            for k in la:
                assert la[k].tobytes() == lb[k].tobytes(), k
    np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(sa, sb)


def test_device_find_batch_validation():
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.finder import find_args
    import torch
    from paper_2402_05396_b200 import build_graph
    g = build_graph([0, 1], [1, 0], [1.0, 2.0], num_nodes=2)
    qv = torch.zeros(4, dtype=torch.int64, device="cuda")
    qt = torch.full((4,), 3.0, dtype=torch.float64, device="cuda")
    a1 = find_args(qv, qt, 3, "recent", 0)
    a2 = find_args(qv, qt, 4, "recent", 0)
    arr = (_lib.tg_find_args * 2)(a1, a2)
    with pytest.raises(ValueError, match="same m and policy"):
        _lib.check(_lib.lib.tg_find_batch(g.c_graph(), arr, 2, None, _lib.stream_ptr()))


@pytest.mark.parametrize("d", [100, 172, 266])
def test_device_node_rows_times_zero_through_gather4(d, monkeypatch):
    """Padded node slots are row(ids) * 0.0 (training.py:227-229): signed
    zeros, inf -> NaN, NaN stays NaN -- the TMA row gather fixes them up in
    shared memory before the store."""
    import torch
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.graph import feat_store, padded_rows, row_pitch
    rng = np.random.default_rng(d)
    V = 3000  # small: the gather4 path is forced with its table-size threshold at 0
    monkeypatch.setenv("TG_K5_G4_MIN_MB", "0")
    table = padded_rows((V,), d, "cuda")
    host = rng.normal(size=(V, d)).astype(np.float32)
    host[5, :3] = [np.inf, -np.inf, np.nan]
    table.copy_(torch.as_tensor(host).cuda())
    n = 5000
    ids = torch.as_tensor(rng.integers(0, V, n)).cuda()
    ids[:50] = 5
    mask = torch.as_tensor(rng.random(n) < 0.6).cuda()
    mask[:25] = False
    out = padded_rows((n,), d, "cuda")
    _lib.check(_lib.lib.tg_lookup_gather(_lib.ptr(ids), _lib.ptr(mask), n, feat_store(table), None, 1, _lib.ptr(out),
                                         row_pitch(d), _lib.stream_ptr()))
    torch.cuda.synchronize()
    rows = table[ids]
    exp = torch.where(mask[:, None], rows, rows * 0.0)
    got = out.view(torch.int32)
    want = exp.contiguous().view(torch.int32)
    nan = torch.isnan(exp)
    assert torch.equal(torch.isnan(out), nan)
    assert torch.equal(got[~nan], want[~nan])
