"""Worker of test_device_sharded_table_ipc_two_processes (launched by
torch.distributed.run, 2 ranks sharing cuda:0, gloo for the handle exchange).

Each rank owns one shard of a hash-defined edge table, maps the other
rank's shard through CUDA IPC (placement.ShardedTable.from_process_group)
and checks, bit for bit against a dense local table:
  * K5 row gathers of ids spread over both shards (bulk and register paths);
  * a 2-hop mini-batch through the sharded table, before and after the
    epoch boundary fills the replicated hot tier.
"""

import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    from paper_2402_05396_b200 import MiniBatchGenerator, _lib
    from paper_2402_05396_b200.graph import row_pitch
    from paper_2402_05396_b200.pipeline import PathConfig
    from paper_2402_05396_b200.shapes import SHAPES, feature_seeds, make_graph, sharded_features, \
        synth_features_device

    E, d = 20011, 186
    tab = sharded_features(E, d, 77)
    dense = synth_features_device(E, d, 77)
    assert tab.world == 2 and len(tab._mapped) == 1
    rng = np.random.default_rng(rank)
    ids = torch.as_tensor(rng.integers(0, E, 5000)).cuda()
    mask = torch.as_tensor(rng.random(5000) < 0.8).cuda()
    exp = torch.where(mask[:, None], dense[ids], torch.zeros((), device="cuda"))
    for register in (False, True):
        if register:
            os.environ["TG_K5_REGISTER_PATH"] = "1"
        else:
            os.environ.pop("TG_K5_REGISTER_PATH", None)
        out = torch.empty((5000, row_pitch(d)), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib.tg_gather_rows(_lib.ptr(ids), _lib.ptr(mask), 5000, tab.c_store(), None, 0,
                                           _lib.ptr(out), row_pitch(d), _lib.stream_ptr()))
        torch.cuda.synchronize()
        assert torch.equal(out[:, :d].view(torch.int32), exp.view(torch.int32)), f"rank {rank} register={register}"
    os.environ.pop("TG_K5_REGISTER_PATH", None)

    spec = SHAPES["E"].scaled(0.0002)
    gd = make_graph(spec, seed=6)
    gs = make_graph(spec, seed=6, edge_placement="sharded")
    assert gs.edge_features.world == 2
    cfg = PathConfig(aggregator="tgat", finder_policy="recent", adaptive_neighbor=False, n=10, batch_size=100)
    a, b = MiniBatchGenerator(gd, cfg, seed=0), MiniBatchGenerator(gs, cfg, seed=0)
    its = [rank, a.iters_per_epoch // 2, a.iters_per_epoch - 1 - rank]
    for epoch in range(2):
        for it in its:
            n, t = (torch.as_tensor(x).cuda() for x in a.roots_for_iteration(it))
            ra = [_lib.torch().clone(r["edge_rows"]) for r in a.generate(n, t, it)]
            rb = [r["edge_rows"] for r in b.generate(n, t, it)]
            for x, y in zip(ra, rb):
                assert torch.equal(x.view(torch.int32), y.view(torch.int32)), (rank, epoch, it)
        a.end_epoch()
        b.end_epoch()
    assert b.cache.resident_count > 0
    torch.cuda.synchronize()
    dist.barrier()
    tab.close()
    gs.edge_features.close()
    dist.barrier()
    print(f"sharded-ipc ok rank {rank}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
