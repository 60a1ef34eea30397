"""Root sharding across ranks (world_size 2, gloo, CPU): the partition and
global-row-key logic of paper_2402_05396_b200/shard.py, run through the CPU
oracle on each rank, reassembles bit-exactly into the 1-rank mini-batch, and
the epoch-boundary all_reduce of cache counters gives the 1-rank counters
and resident set.  The GPU path consumes the same LayerRows (tg_rowmap)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = {
    "B": ("B", 0.004, dict(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=False, n=10), 48),
    "E": ("E", 0.00002, dict(aggregator="tgat", finder_policy="recent", adaptive_neighbor=False, n=10), 64),
    "D": ("D", 0.001, dict(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=True, decoder="gatv2",
                           m=12, n=5, enc_dim=8), 16),
    "C": ("D", 0.001, dict(aggregator="graphmixer", finder_policy="recent", adaptive_neighbor=True,
                           decoder="linear", m=10, n=4, enc_dim=8), 24),
}


def _setup(tag):
    from oracle import shapes as oshapes
    from oracle.pipeline import OracleMiniBatch
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES
    key, f, kw, batch = CASES[tag]
    spec = SHAPES[key].scaled(f)
    cfg = PathConfig(batch_size=batch, cache_fraction=0.2, **kw)
    og = oshapes.make_graph(spec, seed=3)
    return og, cfg, OracleMiniBatch(og, cfg, seed=1)


KEYS = ("sel_ids", "sel_eids", "sel_dts", "sel_mask")


def _worker(rank, world, port, tag, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2402_05396_b200.shard import epoch_allreduce, layer_rows, root_partition
    og, cfg, ob = _setup(tag)
    its = [0, ob.iters_per_epoch // 2, ob.iters_per_epoch - 1]
    shards = []
    for it in its:
        nodes, times = ob.roots_for_iteration(it)
        R1 = nodes.shape[0]
        a, b = root_partition(R1, rank, world)
        w = cfg.n if cfg.adaptive_neighbor else cfg.n
        rows = layer_rows(R1, w, a, b, ob.L)
        recs = ob.generate(nodes[a:b], times[a:b], it,
                           layer_rows=[(r.split, r.base0, r.base1, r.B_global) for r in rows])
        shards.append([{k: r[k] for k in KEYS + (("edge_rows",) if r.get("edge_rows") is not None else ())}
                       for r in recs])
    counters = torch.as_tensor(ob.cache.counters.copy())
    stats = torch.as_tensor(np.array(ob.cache.epochs[-1], dtype=np.int64))
    epoch_allreduce([counters, stats])
    gathered = [None] * world
    dist.all_gather_object(gathered, shards)
    if rank == 0:
        import pickle
        with open(out, "wb") as fh:
            pickle.dump((gathered, counters.numpy(), stats.numpy()), fh)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _reassemble(parts, R1, w, world, layer_index):
    """Concatenate shard outputs into the 1-rank layout; hop-2 rows are
    [targets of all shards || children of all shards] (training.py:312)."""
    if layer_index == 0:
        return np.concatenate(parts)
    from paper_2402_05396_b200.shard import root_partition
    tg, ch = [], []
    for r, p in enumerate(parts):
        a, b = root_partition(R1, r, world)
        nb = b - a
        tg.append(p[:nb])
        ch.append(p[nb:])
    return np.concatenate(tg + ch)


@pytest.mark.parametrize("tag", list(CASES))
def test_root_sharded_minibatch_equals_single_rank(tag, tmp_path):
    import pickle
    world = 2
    path = str(tmp_path / "shards.pkl")
    mp.start_processes(_worker, args=(world, _free_port(), tag, path), nprocs=world, start_method="spawn", join=True)
    with open(path, "rb") as fh:
        gathered, counters, stats = pickle.load(fh)
    og, cfg, ob = _setup(tag)
    its = [0, ob.iters_per_epoch // 2, ob.iters_per_epoch - 1]
    for k, it in enumerate(its):
        nodes, times = ob.roots_for_iteration(it)
        full = ob.generate(nodes, times, it)
        for li, rec in enumerate(full):
            for key in KEYS + (("edge_rows",) if rec.get("edge_rows") is not None else ()):
                got = _reassemble([gathered[r][k][li][key] for r in range(world)], nodes.shape[0], cfg.n, world, li)
                assert got.tobytes() == np.ascontiguousarray(rec[key]).tobytes(), (tag, it, li, key)
    np.testing.assert_array_equal(counters, ob.cache.counters)
    assert list(stats) == ob.cache.epochs[-1]
    # identical replacement on every rank follows from identical counters
    assert ob.cache.maybe_replace() in (True, False)
