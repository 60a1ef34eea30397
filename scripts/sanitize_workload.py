"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
smoke() (2-hop uniform + cache, adaptive gatv2 on the tensor cores, WOR),
a GraphMixer-linear adaptive batch (LN-fused GEMMs, token mixer), the epoch
boundary (K6 replacement) and one K9 selection."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402
from oracle import shapes as oshapes  # noqa: E402
from paper_2402_05396_b200 import MiniBatchGenerator, build_graph  # noqa: E402
from paper_2402_05396_b200.pipeline import PathConfig  # noqa: E402
from paper_2402_05396_b200.shapes import SHAPES  # noqa: E402

__graft_entry__.smoke()
spec = SHAPES["C"].scaled(0.0004)
og = oshapes.make_graph(spec, seed=4)
g = build_graph(og.src, og.dst, og.ts, num_nodes=og.num_nodes, edge_features=og.edge_features)
cfg = PathConfig(aggregator="graphmixer", adaptive_neighbor=True, m=25, n=10, batch_size=40, precision="float32",
                 adaptive_minibatch=True)
gen = MiniBatchGenerator(g, cfg, seed=2)
for it in (1, gen.iters_per_epoch // 2):
    n, t = gen.roots_for_iteration(it)
    recs = gen.generate(torch.as_tensor(n).cuda(), torch.as_tensor(t).cuda(), it)
torch.cuda.synchronize()
gen.end_epoch()
sel = gen.select_roots(3) if hasattr(gen, "select_roots") else None
# hub windows through the coarse time index (K2), uniform and recent
from paper_2402_05396_b200 import batch_find_arrays  # noqa: E402
rng = np.random.default_rng(0)
hub = build_graph(rng.integers(0, 40, 200_000), rng.integers(0, 40, 200_000),
                  np.sort(np.floor(rng.random(200_000) * 25_000)), num_nodes=40)
for policy in ("recent", "uniform"):
    batch_find_arrays(hub, rng.integers(0, 40, 4000), rng.random(4000) * 26_000, 10, policy=policy, seed=1)
torch.cuda.synchronize()
print("sanitize workload done:", int(recs[0]["sel_mask"].sum()), "selected;", "select_roots" if sel is not None else "")
