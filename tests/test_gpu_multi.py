"""Graph-replayed steps and the multi-rank bench.

* ``StepGraph`` (CUDA-graph replay of G steps, seeds read from device
  memory through ``tg_find_args.seed_ptr``) reproduces ``generate`` bit for
  bit, for whole batches and for a root shard with global row keys, and
  counts the cache exactly like it.
* ``bench.py --gpus 2`` self-launches two ranks (here both on cuda:0 over
  gloo, ``TG_BENCH_SHARE_GPU=1``), splits every batch's roots between them,
  and each rank's block is bit-exact against the CPU oracle run with the
  same global row keys -- i.e. the union of the shards is the 1-GPU batch.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("sel_ids", "sel_eids", "sel_dts", "sel_mask", "next_v", "next_t", "edge_rows")


def _np(x):
    return x.detach().cpu().numpy()


def _graph(policy, seed=2):
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["E"].scaled(0.0002)
    og = oshapes.make_graph(spec, seed=seed)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
    cfg = PathConfig(aggregator="tgat", finder_policy=policy, adaptive_neighbor=False, n=10, batch_size=96)
    return g, cfg, (lambda: MiniBatchGenerator(g, cfg, seed=0))


@pytest.mark.parametrize("policy,G,world", [("recent", 1, 1), ("uniform", 2, 1), ("uniform", 2, 3),
                                            ("recent", 3, 2)])
def test_step_graph_matches_generate(policy, G, world):
    import torch
    from paper_2402_05396_b200.pipeline import StepGraph
    from paper_2402_05396_b200.shard import layer_rows, root_partition
    g, cfg, make = _graph(policy)
    ref_gen, gr_gen = make(), make()
    its = list(range(0, ref_gen.iters_per_epoch, max(1, ref_gen.iters_per_epoch // 7)))[:2 * G]
    rank = world - 1
    host, refs = [], []
    for it in its:
        n, t = ref_gen.roots_for_iteration(it)
        R1 = n.shape[0]
        a, b = root_partition(R1, rank, world)
        lr = layer_rows(R1, cfg.n, a, b, ref_gen.L) if world > 1 else None
        host.append((n[a:b], t[a:b], ref_gen.seeds_for(it), lr))
        recs = ref_gen.generate(torch.as_tensor(n[a:b]).cuda(), torch.as_tensor(t[a:b]).cuda(), it, layer_rows=lr)
        refs.append([{k: _np(r[k]) for k in KEYS if k in r} for r in recs])
    sg = StepGraph(gr_gen, int(host[0][0].shape[0]), key="t", G=G, layer_rows=host[0][3])
    rows = torch.as_tensor(np.stack([sg.pack(h[0], h[1], h[2]) for h in host])).cuda()
    for i in range(0, len(its), G):
        recs_g = sg.replay(rows[i:i + G])
        torch.cuda.synchronize()
        for j in range(G):
            for ra, rb in zip(refs[i + j], recs_g[j]):
                for k, v in ra.items():
                    assert _np(rb[k]).tobytes() == v.tobytes(), (i + j, rb["layer"], k)
    np.testing.assert_array_equal(_np(ref_gen.cache.counters), _np(gr_gen.cache.counters))
    np.testing.assert_array_equal(_np(ref_gen.cache.stats), _np(gr_gen.cache.stats))


def test_step_graph_rejects_adaptive():
    from oracle import shapes as oshapes
    from paper_2402_05396_b200 import MiniBatchGenerator, build_graph
    from paper_2402_05396_b200.pipeline import PathConfig, StepGraph
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES["D"].scaled(0.001)
    og = oshapes.make_graph(spec, seed=5)
    g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, node_features=og.node_features,
                    edge_features=og.edge_features)
    cfg = PathConfig(aggregator="tgat", finder_policy="uniform", adaptive_neighbor=True, decoder="gatv2", m=12, n=5,
                     batch_size=16, precision="float32")
    with pytest.raises(ValueError):
        StepGraph(MiniBatchGenerator(g, cfg, seed=1), 48, key="x")


def _bench(args, env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, out.stdout[-2000:] + out.stderr[-2000:]
    return json.loads(lines[-1])


def test_bench_two_ranks_root_sharded_bit_exact():
    """`bench.py --gpus 2` (self-launched ranks, root partition): n_gpus 2,
    every rank's block of every checked step bit-exact vs the oracle."""
    r = _bench(["--gpus", "2", "--workload", "B", "--steps", "6", "--warmup", "3", "--no-cpu", "--no-e2e",
                "--parity-steps", "2"], {"TG_BENCH_SHARE_GPU": "1"})
    assert r["n_gpus"] == 2 and r["run"]["partition"] == "roots"
    assert r["parity"]["ranks_checked"] == 2
    assert r["parity"]["mismatches_all_ranks"] == 0 and r["parity"]["slots_checked_all_ranks"] > 0
    assert r["epoch_boundary"]["allreduce_backend"] == "gloo"
    assert r["gpu_launches"] > 0 and r["value"] > 0


def test_bench_one_gpu_graph_and_generate_agree():
    """The graph-replayed and the generate() step loops count the same
    sampled neighbors per step (same batches, same work)."""
    a = _bench(["--workload", "B", "--steps", "6", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-parity"], {})
    b = _bench(["--workload", "B", "--steps", "6", "--warmup", "3", "--no-cpu", "--no-e2e", "--no-parity",
                "--no-graph"], {})
    assert a["sampled_per_step"] == b["sampled_per_step"]
    assert a["run"]["launch"].startswith("CUDA graph") and b["run"]["launch"].startswith("generate()")
