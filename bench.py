"""Benchmark of the TASER mini-batch-generation hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload E] [--impl ours|reference]

A "step" is one mini-batch generation: batch 600 -> 1,800
roots -> 2-hop neighbor finding with materialisation, hop expansion, cache
accounting and the edge-feature slice of every layer (train mode).  Default
workload: GDELT-shaped E (V 16,682, E 191,290,882, 186-d f32 edge rows in
HBM, 2-hop most-recent 10x10, 20% cache).  Roots per step are real Trainer
batches (chronological train slices + substream negatives) spread across
the epoch.  N>1 (torchrun): every rank holds a replica of the T-CSR and the
table and generates its own batches (weak scaling, no data-path collective).

Timing: W untimed steps, then K steps between barrier+synchronize, CUDA
events on the launching stream, max over ranks.  Inputs (142 GB table,
6 GB T-CSR) are far larger than the 126 MB L2 and the timed batches are
spread over the epoch, so no L2 flush is inserted.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0
# BASELINE.json "metric": value = sampled neighbors/s, plus minibatch_gen_ms and roofline.frac
METRIC = "sampled neighbors/sec + mini-batch gen ms (1/2/4/8 B200, % HBM roofline)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--workload", default="E", choices=list("ABCDE"))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-sample", type=float, default=None, help="event fraction of the CPU baseline sample")
    p.add_argument("--cpu-batches", type=int, default=None)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-parity", action="store_true", help="skip the full-size oracle check of timed steps")
    p.add_argument("--parity-steps", type=int, default=None, help="timed steps re-checked (default 3; adaptive 1)")
    p.add_argument("--inflight", type=int, default=None,
                   help="step groups (graphs) in flight; default by root share: 3 (whole batch), 4 (1/2 and less)")
    p.add_argument("--partition", default="roots", choices=["roots", "batches"],
                   help="N>1: split each batch's roots across ranks (north star) or give ranks whole batches")
    p.add_argument("--graph", dest="graph", action="store_true", default=True,
                   help="replay captured CUDA graphs of the step (non-adaptive workloads; default)")
    p.add_argument("--no-graph", dest="graph", action="store_false")
    p.add_argument("--graph-batches", type=int, default=None,
                   help="batches per captured step group; default by root share: 2, 1 (1/2), 2 (1/4), 4 (1/8)")
    p.add_argument("--emulate-shard", default=None, metavar="R/N",
                   help="one process runs rank R's block of an N-way root partition (a scaling projection on one "
                        "GPU; the line is marked emulated)")
    p.add_argument("--placement", default="auto", choices=["auto", "replicated", "sharded"],
                   help="edge-feature placement (placement.py): auto = replicated when the table fits one GPU")
    p.add_argument("--precision", default=None, choices=["float32", "float64"],
                   help="adaptive workloads: the sampler's compute dtype (RunConfig.precision); default float32 "
                        "(tensor cores, q within 1e-5), float64 = the reference's default, bit-exact selections")
    p.add_argument("--trace", default=None, metavar="FILE",
                   help="diagnosis: after the timed passes, replay the step loop under torch.profiler (CUPTI kernel "
                        "timeline, one JSON per kernel: name, stream, start/end us) into FILE; never timed")
    return p.parse_args()


DTYPE = "f64 ts / int64 ids / f32 rows"
DATA = "synthetic (shape generator of SURVEY §8(d), device + bit-identical host twin); random-hash f32 features"


def load_specs():
    """The workload table (paper_2402_05396_b200/specs.py) loaded by file
    path: it has no dependencies, so the reference arm never imports the
    product package nor maps its CUDA library."""
    import importlib.util
    name = "_tg_bench_specs"
    if name not in sys.modules:
        sp = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "paper_2402_05396_b200", "specs.py"))
        mod = importlib.util.module_from_spec(sp)
        sys.modules[name] = mod
        sp.loader.exec_module(mod)
    return sys.modules[name].SHAPES


def workload_config(spec):
    """`config` of both arms: the workload only (runtime facts live elsewhere)."""
    return {"workload": f"{spec.key}:{spec.name}-shaped V={spec.V} E={spec.E} d_e={spec.d_e} d_v={spec.d_v}",
            "path": spec.note, "batch": spec.batch, "roots_per_step": 3 * spec.batch,
            "aggregator": spec.aggregator, "finder_policy": spec.finder_policy, "adaptive": spec.adaptive,
            "cache_fraction": 0.2, "train_mode": True,
            "l2": "inputs larger than L2 (edge table + T-CSR >> 126 MB); timed batches spread over the epoch"}


def step_iterations(S, world, rank, iters):
    """Training iteration of step s: S steps spread over the epoch."""
    return [((s * world + rank) * iters) // (S * world) for s in range(S)]


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured", pk
    except Exception:
        return HBM_FALLBACK_GBS, "fallback", {}


class ClockSampler:
    """NVML poller for SM clock + throttle reasons during a timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    _NAMES = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
              "hw_power_brake_slowdown": 0x80, "sync_boost": 0x10}

    def _sample(self):
        if self.nv is not None:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self._NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.0002)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()
        self._sample()  # the region's last moment (short timed regions see few polls)

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(s)}


# ---------------------------------------------------------------------------
# algorithmic bytes (SURVEY §8(d) formula)
# ---------------------------------------------------------------------------

def layer_bytes(graph, rec, d_e, lookups):
    """Algorithmic bytes of one layer, split into the finder launch (K2+K3:
    search, T-CSR entries, materialised outputs, cache counters) and the row
    gather launch (K5: 4*d_e read per valid slot, 4*d_e written per slot)."""
    import torch
    qv = rec["queries"][0]
    off = graph.tcsr_offsets
    deg = (off[qv + 1] - off[qv]).to(torch.float64)
    probes = torch.ceil(torch.log2(deg + 1.0))
    B = int(qv.shape[0])
    valid = int(rec["sel_mask"].sum().item())
    slots = int(rec["sel_mask"].numel())
    find = 16 * B + 8 * float(probes.sum().item()) + 8 * B + valid * (16 + 24) + (valid * 9 if lookups else 0)
    gather = slots * 4 * d_e + valid * 4 * d_e
    if "q" in rec:  # adaptive: the m candidates' rows are gathered too (training.py:264)
        cvalid = int(rec["mask"].sum().item())
        gather += int(rec["mask"].numel()) * 4 * d_e + cvalid * 4 * d_e
    return {"find": find, "gather": gather, "valid": valid, "slots": slots, "B": B}


def run_ours(args, rank, local_rank, world):
    import numpy as np
    import torch
    import torch.distributed as dist

    # TG_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo (exercises the
    # multi-rank partition / timing / reduction logic on a 1-GPU box; NCCL
    # forbids two ranks on one device).  Normal runs: one rank per GPU, NCCL.
    share = os.environ.get("TG_BENCH_SHARE_GPU") == "1"
    dev_index = 0 if share else local_rank
    torch.cuda.set_device(dev_index)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init lines (nranks) for the record
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    red_dev = "cpu" if share else "cuda"
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.pipeline import MiniBatchGenerator, StepGraph
    from paper_2402_05396_b200.shapes import make_graph
    from paper_2402_05396_b200.shard import epoch_allreduce, layer_rows, root_partition
    from paper_2402_05396_b200.specs import SHAPES

    spec = SHAPES[args.workload]
    partition = args.partition if world > 1 else "roots"
    prank, pworld = rank, world  # whose block of each batch this process generates
    if args.emulate_shard:
        if world > 1:
            raise SystemExit("--emulate-shard is a single-process projection")
        prank, pworld = (int(x) for x in args.emulate_shard.split("/"))
    placement = args.placement
    if placement == "auto":
        # replicate when table + T-CSR + cache state fit in 90% of this GPU's HBM
        need = spec.E * (4 * ((spec.d_e + 3) & ~3) + 2 * 16 + 8 + 24) + spec.V * 8
        total = torch.cuda.get_device_properties(dev_index).total_memory
        placement = "replicated" if need * (world if share else 1) < 0.9 * total else "sharded"
    t0 = time.time()
    g = make_graph(spec, seed=args.seed, edge_placement=placement)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    cfg = spec.path_config(**({"precision": args.precision} if args.precision and spec.adaptive else {}))
    gen = MiniBatchGenerator(g, cfg, seed=0)
    S = args.warmup + args.steps
    iters = gen.iters_per_epoch
    # "roots": every rank works on the SAME global batches and takes a block
    # of each batch's hop-1 roots (north star); "batches":
    # every rank generates its own whole batches (weak-scaling alternative)
    its = step_iterations(S, 1, 0, iters) if partition == "roots" else step_iterations(S, world, rank, iters)
    seeds = [gen.seeds_for(it) for it in its]
    host_roots, roots, lrows, shard = [], [], [], []
    for it in its:
        n, tt = gen.roots_for_iteration(it)
        R1g = int(n.shape[0])
        if partition == "roots" and pworld > 1:
            a, b = root_partition(R1g, prank, pworld)
            lr = layer_rows(R1g, cfg.n, a, b, gen.L)
        else:
            a, b, lr = 0, R1g, None
        shard.append((a, b, R1g))
        lrows.append(lr)
        host_roots.append((n[a:b], tt[a:b]))
        roots.append((torch.as_tensor(n[a:b]).cuda(), torch.as_tensor(tt[a:b]).cuda()))
    stream = torch.cuda.current_stream()
    # smaller root shares are latency-bound: more batches per captured step
    # group and in flight (measured on E, profiles/r02s3_shard_sweep.txt:
    # whole batch 3 x 2, 1/2 share 4 x 1, 1/4 share 4 x 2, 1/8 share 4 x 4);
    # with the 3-tile K5 rings a whole non-adaptive 2-hop batch runs best 2 x 2
    # and the shares 4 x 4 / 3 x 4 (profiles/r02s5_inflight.md: E 60.4 -> 58.7
    # us, B 60.0 -> 56.8 us; 1/2 share 31.1 -> 30.0, 1/4 16.9 -> 16.7, 1/8
    # 10.5 -> 10.1 us)
    kg = {1: (2, 2) if gen.L > 1 and not spec.adaptive else (3, 2), 2: (4, 4)}.get(pworld, (3, 4))
    args.inflight_auto = args.inflight is None
    if args.inflight is None:
        args.inflight = kg[0]
    if args.graph_batches is None:
        args.graph_batches = kg[1]
    K = max(1, args.inflight)

    def step(s, events=None, slot=0):
        return gen.generate(roots[s][0], roots[s][1], its[s], finder_seeds=seeds[s], events=events, slot=slot,
                            layer_rows=lrows[s])

    # the previous epoch (same positive edges, other negatives: it + iters)
    # counts accesses; its epoch boundary -- counters and hit/miss stats
    # summed across ranks (NCCL all_reduce), then K6 on every rank -- fills
    # the cache (cache.py:107-118), so the timed steps see the reference's
    # steady-state resident set (with sharded placement, the hot tier)
    epoch = None
    if gen.cache is not None:
        for s in range(S):
            pn, pt = gen.roots_for_iteration(its[s] + iters)
            a, b, _ = shard[s]
            gen.generate(torch.as_tensor(pn[a:b]).cuda(), torch.as_tensor(pt[a:b]).cuda(), its[s] + iters,
                         layer_rows=lrows[s])
        gen.join()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        from paper_2402_05396_b200.cache import maybe_replace
        t_ar = time.perf_counter()
        epoch_allreduce([gen.cache.counters_i32, gen.cache.stats])
        torch.cuda.synchronize()
        ar_s = time.perf_counter() - t_ar
        t_rp = time.perf_counter()
        replaced = maybe_replace(gen.cache)
        torch.cuda.synchronize()
        rp_s = time.perf_counter() - t_rp
        nbytes = gen.cache.counters_i32.numel() * 4 + gen.cache.stats.numel() * 8
        epoch = {"allreduce_ms": round(ar_s * 1e3, 3), "allreduce_bytes": int(nbytes),
                 "allreduce_backend": dist.get_backend() if world > 1 else None,
                 "allreduce_GB/s": round(nbytes / ar_s / 1e9, 1) if world > 1 else None,
                 "replace_ms": round(rp_s * 1e3, 3), "replaced": bool(replaced),
                 "note": "epoch boundary (training.py:442-443): per-edge int32 counters + hit/miss summed across "
                         "ranks, then K6 top-k replacement on every rank (identical resident sets)"}
        gen.cache.stats.zero_()

    # accounting pass: algorithmic bytes + sampled neighbors of every step
    # (untimed); sharded placement: rows read from a peer's shard (NVLink)
    sharded = hasattr(g.edge_features, "c_store")
    acct = []
    for s in range(S):
        recs = step(s)
        per = [layer_bytes(g, r, g.d_e, gen.cache is not None) for r in recs]
        for p_, r in zip(per, recs):
            p_["sampled"] = int(r["sel_mask"].sum().item())
            p_["peer_rows"] = 0
            if sharded and "edge_rows" in r:
                e, mk = r["sel_eids"].flatten(), r["sel_mask"].flatten()
                miss = mk & (gen.cache.slot_of[e] < 0) if gen.cache is not None else mk
                own = (e // g.edge_features.shard_rows) == g.edge_features.rank
                p_["peer_rows"] = int((miss & ~own).sum().item())
        acct.append(per)
    torch.cuda.synchronize()

    # CUDA-graph replay (non-adaptive paths): G batches per graph, K graphs
    # in flight; falls back to generate() when the steps' root counts differ
    R1s = {int(r[0].shape[0]) for r in roots}
    use_graph = args.graph and not spec.adaptive and len(R1s) == 1
    graphs, packed, G = [], None, max(1, args.graph_batches)
    launches_per_step = None
    graph_at = {}
    if use_graph:
        # one graph per group of G consecutive steps, reading that group's
        # packed inputs in place (a replay is one graph launch, no copy);
        # groups cycle over K streams / workspace slots (K groups in flight)
        R1 = R1s.pop()
        gstreams = [torch.cuda.Stream() for _ in range(K)]
        rows = np.stack([StepGraph.pack_row(R1, gen.L, host_roots[s][0], host_roots[s][1], seeds[s])
                         for s in range(S)])
        packed = torch.as_tensor(rows).cuda()
        c0 = _lib.launch_count()
        for lo_, hi_ in ((0, args.warmup), (args.warmup, S)):
            for gi, s0 in enumerate(range(lo_, hi_ - G + 1, G)):
                graph_at[s0] = StepGraph(gen, R1, key=("bench", gi % K), G=G, layer_rows=lrows[0],
                                         inputs=packed[s0:s0 + G], stream=gstreams[gi % K])
        launches_per_step = (_lib.launch_count() - c0) / (2 * G * max(1, len(graph_at)))  # priming + capture
        graphs = list(graph_at.values())

    def run_steps(lo, hi):
        """Steps [lo, hi) as the data loader runs them (graph groups of G,
        K in flight; the remainder through generate())."""
        if use_graph:
            for gs in gstreams:
                gs.wait_stream(stream)
            s = lo
            while s + G <= hi and s in graph_at:
                graph_at[s].launch_bound()
                s += G
            for gs in gstreams:
                stream.wait_stream(gs)
            for r in range(s, hi):
                step(r)
        else:
            # private slot streams 1..K (slot 0 is the caller's stream, which
            # every slot waits on for its roots, so it must not carry batches)
            for k in range(1, K + 1):
                gen.slot_stream(k).wait_stream(stream)
            for r in range(lo, hi):
                step(r, slot=1 + r % K)
            gen.join(stream)

    # warm-up
    run_steps(0, args.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # timed pass A: the step loop as a data loader runs it
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        h0 = time.perf_counter()
        run_steps(args.warmup, S)
        e1.record(stream)
        host_enqueue_ms = (time.perf_counter() - h0) * 1e3
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - launches0
    if use_graph:
        n_graph = (args.steps // G) * G
        launches += int(round(launches_per_step * n_graph))
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
    sampled = sum(sum(p["sampled"] for p in acct[s]) for s in range(args.warmup, S))
    peer = sum(sum(p["peer_rows"] for p in acct[s]) for s in range(args.warmup, S))
    samp_t = torch.tensor([float(sampled), float(peer)], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(samp_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    total_sampled = float(samp_t[0].item())
    total_peer_rows = float(samp_t[1].item())
    value = total_sampled / (ms_max / 1e3)

    if args.trace and rank == 0:
        trace_steps(args.trace, lambda: run_steps(args.warmup, S))

    # timed pass A1: single-batch latency ("mini-batch gen ms"):
    # the same steps through generate() with ONE batch in flight
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0.record(stream)
    for s in range(args.warmup, S):
        step(s, slot=0)
    gen.join(stream)
    l1.record(stream)
    torch.cuda.synchronize()
    lat_t = torch.tensor([l0.elapsed_time(l1) / args.steps], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(lat_t, op=dist.ReduceOp.MAX)
    gen_ms = float(lat_t.item())

    # timed pass B: per-launch events for the roofline of the fused kernel
    L = gen.L
    evs = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(L)] for _ in range(S)]
    sev = [[tuple(torch.cuda.Event(enable_timing=True) for _ in range(2)) for _ in range(L)] for _ in range(S)]
    torch.cuda.synchronize()
    wsl = gen.workspace(int(roots[0][0].shape[0]), 0).layers
    for s in range(args.warmup, S):
        if spec.adaptive:
            for li, rec in enumerate(wsl):
                rec["score_events"] = sev[s][li]
        step(s, events=evs[s])
    for rec in wsl:
        rec.pop("score_events", None)
    torch.cuda.synchronize()
    f_ms, g_ms = [0.0] * L, [0.0] * L
    f_by, g_by = [0.0] * L, [0.0] * L
    for s in range(args.warmup, S):
        for li in range(L):
            e_start, e_end, e_mid = evs[s][li]
            f_ms[li] += e_start.elapsed_time(e_mid)
            g_ms[li] += e_mid.elapsed_time(e_end)
            f_by[li] += acct[s][li]["find"]
            g_by[li] += acct[s][li]["gather"]
    peak, peak_kind, peaks = load_peaks()
    gms, gby = sum(g_ms), sum(g_by)
    fms, fby = sum(f_ms), sum(f_by)
    achieved = gby / (gms / 1e3) / 1e9
    n_launch = args.steps * L
    # non-adaptive layers: one K5 launch per step carries every layer's rows
    merged = not spec.adaptive and gen.merge_gathers and L > 1
    g_launch = args.steps if merged else n_launch
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as fh:
                tr = json.load(fh)
            if tr.get("workload") == args.workload:
                traffic = tr.get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    by_t = torch.tensor([gby + fby], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(by_t, op=dist.ReduceOp.SUM)
    job_bytes = float(by_t.item())
    roofline = {"bound": "hbm", "kernel": "K5 edge-row slice on the TMA engine (tg::row_gather_g4_kernel: tile::gather4, "
                                          "4 table rows per request; per-row bulk copies with a hot tier / peer shards), "
                                          "dominant" + ("; every layer's rows in one launch per step" if merged else ""),
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else
                f"fallback {HBM_FALLBACK_GBS} GB/s (B200_PROFILING.md)",
                "traffic": traffic if world == 1 else None,
                "scope": "rank 0's launches" if world > 1 else "the launches of the run",
                "algorithmic_bytes_per_launch": round(gby / g_launch),
                "avg_launch_us": round(gms / g_launch * 1e3, 2),
                "finder": {"kernel": "tg::find_kernel (K2+K3)", "avg_launch_us": round(fms / n_launch * 1e3, 2),
                           "algorithmic_bytes_per_launch": round(fby / n_launch),
                           "GB/s": round(fby / (fms / 1e3) / 1e9, 1)},
                "path": {"bytes_per_step": round(job_bytes / args.steps),
                         "GB/s_over_step": round(job_bytes / (ms_max / 1e3) / 1e9, 1),
                         "peak": round(peak * world, 1),
                         "frac_over_step": round(job_bytes / (ms_max / 1e3) / 1e9 / (peak * world), 4),
                         "scope": f"all ranks' algorithmic bytes / the slowest rank's timed region, against "
                                  f"{world} x the 1-GPU peak"},
                "per_layer": [{"layer": gen.L - li, "roots": acct[args.warmup][li]["B"],
                               "find_us": round(f_ms[li] / args.steps * 1e3, 2),
                               "gather_us": round(g_ms[li] / args.steps * 1e3, 2),
                               "gather_GB/s": round(g_by[li] / (g_ms[li] / 1e3) / 1e9, 1) if not merged else None,
                               "gather_bytes": round(g_by[li] / args.steps)} for li in range(L)],
                "per_layer_note": "merged K5: the last layer's gather_us is the one launch moving every layer's rows"
                                  if merged else None,
                "share_of_step": round(gms / max(ms, 1e-9), 3)}

    if spec.adaptive:
        # adaptive workloads: the dominant kernel is K7 scoring (tensor-bound)
        model = gen._adaptive.model
        k7_ms = sum(sev[s][li][0].elapsed_time(sev[s][li][1]) for s in range(args.warmup, S) for li in range(L))
        k7_flops = sum(model.flops(acct[s][li]["B"]) for s in range(args.warmup, S) for li in range(L))
        tf32_peak, tf32_src = tf32_peak_tflops(peaks)
        ach = k7_flops / (k7_ms / 1e3) / 1e12
        k7 = {"bound": "tensor", "kernel": "K7 tg_score: tcgen05 3xTF32 GEMMs (tc_gemm_kernel) + encoders, token "
                                           "mixer, decoder, masked softmax",
              "achieved": round(ach, 2), "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
              "frac": round(ach / tf32_peak, 4), "traffic": None,
              "peak_source": tf32_src + ("; achieved counts useful FLOPs -- the 3xTF32 split issues 3 tf32 MMAs per "
                                         "product, so 1/3 is the ceiling" if model.tensor_cores
                                         else "; FFMA path (trans decoder)"),
              "precision": model.precision, "tensor_cores": model.tensor_cores,
              "avg_us_per_layer": round(k7_ms / (args.steps * L) * 1e3, 2),
              "flops_per_step": round(k7_flops / args.steps), "share_of_step": round(k7_ms / max(ms, 1e-9), 3),
              "hbm": {"scope": "whole step: all algorithmic bytes (finder, candidate + selected rows) / step time",
                      "achieved": roofline["path"]["GB/s_over_step"], "peak": roofline["path"]["peak"],
                      "unit": "GB/s", "frac": roofline["path"]["frac_over_step"]}}
        roofline = k7

    hit_rate = None
    if gen.cache is not None:
        hm = gen.cache.stats.to(red_dev, torch.float64)
        if world > 1:
            dist.all_reduce(hm, op=dist.ReduceOp.SUM)
        hm = hm.tolist()
        hit_rate = round(hm[0] / max(1, hm[0] + hm[1]), 4)

    # bit-exactness of timed steps at the full workload size (untimed): rank 0
    # checks its own block of roots (global RNG keys) against the oracle
    # (every rank when the graph is small enough for N host copies; the
    # per-rank mismatch counts are summed)
    parity = None
    par_all = spec.E <= 50_000_000
    if not args.no_parity and (rank == 0 or par_all):
        n_chk = args.parity_steps if args.parity_steps is not None else (1 if spec.adaptive else 3)
        n_chk = max(1, min(n_chk, args.steps))
        chk = sorted({args.warmup + (i * (args.steps - 1)) // max(1, n_chk - 1) for i in range(n_chk)})
        parity = parity_check(args, spec, g, gen, its, roots, seeds, chk, lrows)
    if world > 1:
        if not args.no_parity and par_all:
            mm = torch.tensor([float(parity["mismatches"]), float(parity["slots_checked"])], device=red_dev,
                              dtype=torch.float64)
            dist.all_reduce(mm, op=dist.ReduceOp.SUM)
            if rank == 0:
                parity.update(ranks_checked=world, mismatches_all_ranks=int(mm[0].item()),
                              slots_checked_all_ranks=int(mm[1].item()))
        dist.barrier()

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, gen, its, seeds, acct, world, dist, red_dev, host_roots, lrows)

    nvlink = None
    if sharded:
        pb = total_peer_rows * 4 * g.d_e
        nvlink = {"peer_row_bytes_per_step": round(pb / args.steps),
                  "GB/s_per_gpu": round(pb / world / (ms_max / 1e3) / 1e9, 1), "peak_per_gpu": 900.0,
                  "frac": round(pb / world / (ms_max / 1e3) / 1e9 / 900.0, 4),
                  "note": "cache misses whose eid lives in another rank's shard, read by K5 over NVLink P2P"}
    desc = {"roots": f"root-sharded x{world}: every rank takes a block of each batch's hop-1 roots (global RNG "
                     f"keys, replicated T-CSR, {placement} edge table)",
            "batches": f"batch-sharded x{world}: every rank generates its own whole batches (replicated T-CSR, "
                       f"{placement} edge table)"}[partition]
    result = {
        "metric": METRIC,
        "value": round(value, 1), "unit": "sampled neighbors/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong" if (partition == "roots" and world > 1) else "weak",
        "vs_baseline": None, "dtype": DTYPE, "data": DATA,
        "config": dict(workload_config(spec), **({"sampler_precision": cfg.precision} if spec.adaptive else {})),
        "parallelism": desc,
        "run": {"partition": partition, "edge_placement": placement, "cache_hit_rate": hit_rate,
                "inflight": K, "host_enqueue_ms_per_step": round(host_enqueue_ms / args.steps, 4), "launch": f"CUDA graph replay, {G} batch(es) per graph, {K} graphs in flight"
                if use_graph else f"generate() per batch, {K} slots in flight",
                "graph_build_s": round(build_s, 2), "shared_gpu": share},
        "sampled_per_step": round(total_sampled / args.steps, 1),
        "minibatch_gen_ms": round(gen_ms, 4),
        "minibatch_gen_ms_note": "single-batch latency: device roots -> every buffer of the step ready, one batch "
                                 "in flight through generate() (ms_per_step is the steady state)",
        "gpu_launches": int(launches),
        "roofline": roofline,
        "clocks": clk.summary(),
        "e2e": e2e,
        "parity": parity,
        "epoch_boundary": epoch,
        "nvlink": nvlink,
    }
    if args.emulate_shard:
        result["emulated_shard"] = {"rank": prank, "world": pworld,
                                    "note": "this process generated only its block of every batch; value is that "
                                            "block's throughput (a per-rank rate, not a whole-job number)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(args, spec, value_unit="sampled neighbors/s")
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def trace_steps(path, fn):
    """Kernel timeline of fn() from CUPTI (torch.profiler), for overlap
    diagnosis only: one JSON line per kernel with its stream and start / end
    (us, relative to the first kernel)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    tmp = path + ".chrome.json"
    prof.export_chrome_trace(tmp)
    with open(tmp) as fh:
        ev = json.load(fh)
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    t0 = min(e["ts"] for e in ks) if ks else 0
    with open(path, "w") as fh:
        for e in sorted(ks, key=lambda e: e["ts"]):
            fh.write(json.dumps({"name": e["name"][:80], "stream": e.get("args", {}).get("stream", e.get("tid")),
                                 "start": round(e["ts"] - t0, 2), "end": round(e["ts"] - t0 + e["dur"], 2)}) + "\n")
    os.remove(tmp)


def tf32_peak_tflops(peaks):
    """Dense TF32 tensor peak: MEASURED_PEAKS.json tf32_tflops when the driver
    measured it, else profiles/tf32_peak.json (this repo's own 1xTF32
    tcgen05 GEMM at 8192^3, scripts/tf32_peak.py), else bf16 / 2."""
    if "tf32_tflops" in peaks:
        return float(peaks["tf32_tflops"]), "measured (MEASURED_PEAKS.json tf32_tflops)"
    path = os.path.join(ROOT, "profiles", "tf32_peak.json")
    if os.path.exists(path):
        try:
            with open(path) as fh:
                pk = json.load(fh)
            return float(pk["tf32_tflops"]), f"measured ({pk.get('how', 'profiles/tf32_peak.json')})"
        except Exception:
            pass
    bf16 = float(peaks.get("bf16_tflops", 1647.8))
    return 0.5 * bf16, "estimate: measured bf16_tflops x 0.5 (dense TF32 rate)"


def parity_check(args, spec, g, gen, its, roots, seeds, steps, lrows=None):
    """Bit-exactness of timed steps at the FULL workload size, against the CPU
    oracle (oracle/, pinned to the reference's goldens), outside the timed
    regions.  Host copies of the device events and T-CSR; the T-CSR is checked
    entry by entry against graph.py:94-152's definition (oracle.tcsr.check_tcsr);
    each checked step is re-generated (slot 0) and compared with the oracle's
    mini-batch for the same roots: per layer sel_ids / sel_eids / sel_dts /
    sel_mask, the next hop's queries, every edge row (bytes; rows regenerated
    from the feature hash for the eids the step read), and the step's cache
    accounting (per-edge counter increments, hit/miss) against the oracle cache
    holding the device's resident set.  Adaptive layers: candidates bit-exact,
    q within 1e-5 relative (the north star's fp32 bound), selections counted.
    Root-sharded runs: this rank's block of roots with its global row keys
    (lrows), which the oracle takes as layer_rows."""
    import numpy as np
    import torch
    from types import SimpleNamespace
    from oracle import shapes as oshapes
    from oracle.pipeline import OracleMiniBatch
    from oracle.tcsr import OracleGraph, check_tcsr
    t0 = time.time()
    h = lambda x: x.cpu().numpy()  # noqa: E731
    src, dst, ts = h(g.src), h(g.dst), h(g.ts)
    off, nbr, tts, eid = h(g.tcsr_offsets), h(g.nbr32), h(g.tcsr_ts), h(g.eid32)
    res = {"workload": workload_config(spec)["workload"], "oracle": "oracle/ (numpy + numba restatement pinned to "
                                                                   "golden vectors of the real reference)"}
    # events: the device generator vs its host twin at 1M sampled eids
    rs = np.random.default_rng(7).integers(0, spec.E, size=min(spec.E, 1 << 20))
    es, ed, et = oshapes.synth_events_at(spec.V, spec.E, args.seed, rs)
    ev_bad = int((es != src[rs]).sum() + (ed != dst[rs]).sum() + (et.view(np.int64) != ts[rs].view(np.int64)).sum())
    tc_bad, n_entries = check_tcsr(src, dst, ts, off, nbr, tts, eid)
    res.update(events_checked=int(rs.size), event_mismatches=ev_bad, tcsr_entries_checked=n_entries,
               tcsr_mismatches=tc_bad)
    eseed, nseed = oshapes.feature_seeds(args.seed)
    og = OracleGraph(num_nodes=g.num_nodes, src=src, dst=dst, ts=ts, tcsr_offsets=off, tcsr_neighbors=nbr,
                     tcsr_ts=tts, tcsr_eids=eid,
                     node_features=oshapes.synth_features(0, spec.V, spec.d_v, nseed) if spec.d_v else None,
                     edge_features=oshapes.HashRows(spec.E, spec.d_e, eseed) if spec.d_e else None)
    cfg = SimpleNamespace(**vars(gen.cfg))
    ob = OracleMiniBatch(og, cfg, seed=gen.seed, dtype=np.float32)
    mism, slots, rows_checked, q_err, sel_rows_diff = 0, 0, 0, 0.0, 0
    skipped_layers, cache_skipped = 0, 0
    detail = []
    cache = gen.cache
    for s in steps:
        if cache is not None:
            torch.cuda.synchronize()
            c0, st0 = cache.counters_i32.clone(), cache.stats.clone()
            ob.cache.resident = h(cache.slot_of >= 0)
            ob.cache.counters[:] = 0
            ob.cache.epochs = [[0, 0]]
        lr = lrows[s] if lrows is not None else None
        recs = gen.generate(roots[s][0], roots[s][1], its[s], finder_seeds=seeds[s], layer_rows=lr)
        torch.cuda.synchronize()
        orecs = ob.generate(h(roots[s][0]), h(roots[s][1]), its[s],
                            layer_rows=None if lr is None else [(r.split, r.base0, r.base1, r.B_global) for r in lr])
        # f32 q may move a WOR draw across a cumsum boundary (north star: not
        # bit-exact there); the cache then counts the device's picks instead
        # of the oracle's -- expected counters are adjusted by exactly that
        # difference, and a layer below a differing selection (other
        # queries) is not comparable
        sel_adj, diverged = [], False
        for r, o in zip(recs, orecs):
            if diverged:
                skipped_layers += 1
                continue
            keys = ["ids", "eids", "dts", "mask"] if "q" in r else ["sel_ids", "sel_eids", "sel_dts", "sel_mask"]
            keys += [k for k in ("next_v", "next_t", "edge_rows", "node_rows", "tgt_rows") if k in r and k in o
                     and o[k] is not None and "q" not in r]
            for k in keys:
                got = h(r[k])
                exp = np.asarray(o[k]).astype(got.dtype)
                bad = int((got.view(np.uint8).reshape(got.shape[0], -1) !=
                           exp.view(np.uint8).reshape(exp.shape[0], -1)).any(axis=1).sum())
                if bad:
                    detail.append({"step": int(s), "layer": int(r["layer"]), "key": k, "rows": bad})
                mism += bad
            slots += int(r["sel_mask"].numel())
            if "edge_rows" in keys:
                rows_checked += int(r["sel_mask"].sum())
            if "q" in r:
                q, rq = h(r["q"]).astype(np.float64), o["q"]
                q_err = max(q_err, float(np.max(np.abs(q - rq) / np.maximum(np.abs(rq), 1e-30),
                                                initial=0.0, where=rq > 0)))
                nd = int((h(r["sel_eids"]) != o["sel_eids"]).any(axis=1).sum())
                sel_rows_diff += nd
                if nd:
                    sel_adj.append((h(r["sel_eids"])[h(r["sel_mask"])], o["sel_eids"][o["sel_mask"]]))
                    diverged = int(r["layer"]) > 1
        if cache is not None and diverged:
            cache_skipped += 1
        elif cache is not None:
            torch.cuda.synchronize()
            d = (cache.counters_i32 - c0).to(torch.int64)
            nz = torch.nonzero(d).flatten()
            got_idx, got_val = h(nz), h(d[nz])
            expc = ob.cache.counters.astype(np.int64).copy()
            exps = np.asarray(ob.cache.epochs[-1], dtype=np.int64).copy()
            for dsel, osel in sel_adj:
                np.add.at(expc, dsel, 1)
                np.add.at(expc, osel, -1)
                res = ob.cache.resident
                exps += [int(res[dsel].sum()) - int(res[osel].sum()), int((~res[dsel]).sum()) - int((~res[osel]).sum())]
            exp_idx = np.flatnonzero(expc)
            cbad = int(not (np.array_equal(got_idx, exp_idx) and np.array_equal(got_val, expc[exp_idx])))
            hm = h(cache.stats - st0).astype(np.int64)
            sbad = int(not np.array_equal(hm, exps))
            if cbad or sbad:
                detail.append({"step": int(s), "key": "cache", "counters": cbad, "stats": sbad})
            mism += cbad + sbad
    if lrows is not None and lrows[steps[0]] is not None:
        res["shard"] = f"rank 0's block of {int(roots[steps[0]][0].shape[0])} hop-1 roots (global RNG keys)"
    res.update(steps_checked=len(steps), step_indices=[int(s) for s in steps], slots_checked=slots,
               edge_rows_checked=rows_checked, mismatches=mism, check_s=round(time.time() - t0, 1))
    if spec.adaptive:
        res.update(q_max_rel_err=q_err, q_bound=1e-5, selected_rows_differing=sel_rows_diff,
                   layers_skipped_after_divergence=skipped_layers, cache_checks_skipped=cache_skipped,
                   note="adaptive: candidates / cache bit-exact (cache counts adjusted for rows whose f32 q moved "
                        "a WOR draw across a cumsum boundary); f32 q vs the oracle's f64 q within the bound")
    if detail:
        res["detail"] = detail[:20]
    return res


def run_e2e(args, gen, its, seeds, acct, world, dist, red_dev="cuda", host_roots=None, lrows=None):
    """The user's call with HOST buffers: pinned roots -> device, generate,
    every output of the step (ids/eids/dts/mask per layer + edge rows) back
    into pinned host memory, all inside the timed region.  With --inflight K
    the copies of batch i overlap the generation of batch i+1 (K slots, each
    with its own stream, device roots and pinned output buffers).  Root-sharded
    runs: each rank copies in its block of roots and copies out its rows; the
    byte counts are the whole job's (all ranks) per step."""
    import torch
    S = args.warmup + args.steps
    # the copies dominate this leg (PCIe): it keeps the three slots it was
    # measured with unless --inflight was given (profiles/r02s5_inflight.md)
    K = max(3, args.inflight) if getattr(args, "inflight_auto", False) else max(1, args.inflight)
    if lrows is None:
        lrows = [None] * S
    pinned = []
    for s, it in enumerate(its):
        n, t = host_roots[s] if host_roots is not None else gen.roots_for_iteration(it)
        pinned.append((torch.as_tensor(n).pin_memory(), torch.as_tensor(t).pin_memory()))
    host_roots = pinned
    R1 = int(host_roots[0][0].shape[0])
    dv = [torch.empty(R1, dtype=torch.int64, device="cuda") for _ in range(K)]
    dt = [torch.empty(R1, dtype=torch.float64, device="cuda") for _ in range(K)]
    keys = ("sel_ids", "sel_eids", "sel_dts", "sel_mask", "edge_rows", "node_rows", "tgt_rows")
    recs = gen.generate(dv[0].copy_(host_roots[0][0]), dt[0].copy_(host_roots[0][1]), its[0], finder_seeds=seeds[0],
                        layer_rows=lrows[0])
    host_out = [[{k: torch.empty(r[k].shape, dtype=r[k].dtype).pin_memory() for k in keys if k in r} for r in recs]
                for _ in range(K)]
    d2h = sum(v.numel() * v.element_size() for ho in host_out[0] for v in ho.values())
    h2d = host_roots[0][0].numel() * 8 + host_roots[0][1].numel() * 8

    def one(s):
        k = s % K
        st = gen.slot_stream(k)
        with torch.cuda.stream(st):
            dv[k].copy_(host_roots[s][0], non_blocking=True)
            dt[k].copy_(host_roots[s][1], non_blocking=True)
            out = gen.generate(dv[k], dt[k], its[s], finder_seeds=seeds[s], slot=k, layer_rows=lrows[s])
            for r, ho in zip(out, host_out[k]):
                for key, v in ho.items():
                    v.copy_(r[key], non_blocking=True)

    for s in range(args.warmup):
        one(s)
    gen.join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.current_stream()
    e0.record(stream)
    for k in range(1, K):
        gen.slot_stream(k).wait_stream(stream)
    for s in range(args.warmup, S):
        one(s)
    gen.join(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
    samp = sum(sum(p["sampled"] for p in acct[s]) for s in range(args.warmup, S))
    samp_t = torch.tensor([float(samp), float(h2d), float(d2h)], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(samp_t, op=dist.ReduceOp.SUM)
    h2d, d2h = float(samp_t[1].item()), float(samp_t[2].item())
    return {"value": round(float(samp_t[0].item()) / (float(ms_t.item()) / 1e3), 1), "unit": "sampled neighbors/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(float(ms_t.item()) / args.steps, 4),
            "pcie_GB/s_per_gpu": round((h2d + d2h) / world / (float(ms_t.item()) / args.steps / 1e3) / 1e9, 1),
            "note": f"pinned host roots in, every mini-batch buffer (incl. f32 feature rows) out, per step; "
                    f"{K} batches in flight"}


# ---------------------------------------------------------------------------
# CPU baselines: the oracle port on a bounded sample (our arm's cpu_baseline)
# and the REAL reference (baseline/_ref tgadapt) for --impl reference
# ---------------------------------------------------------------------------

CPU_SAMPLE = {"A": 1.0, "B": 1.0, "C": 0.02, "D": 0.25, "E": 1 / 16}
CPU_BATCHES = {"A": 40, "B": 20, "C": 2, "D": 4, "E": 20}
# reference arm: timed batches are capped for the adaptive shapes, whose f32
# scoring costs seconds per batch on the host (18.7 s at C)
REF_MAX_STEPS = {"A": 1000, "B": 1000, "C": 2, "D": 6, "E": 1000}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(args, spec, value_unit):
    import numpy as np
    from types import SimpleNamespace
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
    from oracle import finder as ofinder
    from oracle import shapes as oshapes
    from oracle.pipeline import OracleMiniBatch
    frac = args.cpu_sample if args.cpu_sample is not None else CPU_SAMPLE[spec.key]
    nb = args.cpu_batches if args.cpu_batches is not None else CPU_BATCHES[spec.key]
    sspec = spec.scaled(frac) if frac < 1.0 else spec
    t0 = time.time()
    og = oshapes.make_graph(sspec, seed=args.seed, features=True)
    build_s = time.time() - t0
    ofinder.set_threads(os.cpu_count())
    fields = sspec.config_fields()
    # RunConfig's decoder default (training.py:82-83), as PathConfig.__post_init__ sets it
    fields.setdefault("decoder", "gatv2" if fields["aggregator"] == "tgat" else "linear")
    cfg = SimpleNamespace(**fields, cache_epsilon=None, window=None, split_ratios=(0.6, 0.2, 0.2),
                          enc_dim=100, time_span=None)
    ob = OracleMiniBatch(og, cfg, seed=0)
    iters = ob.iters_per_epoch
    its = [(s * iters) // (nb + 2) for s in range(nb + 2)]
    # JIT warm-up on the first two batches
    for it in its[:2]:
        n, t = ob.roots_for_iteration(it)
        ob.generate(n, t, it)
    sampled = 0
    t0 = time.perf_counter()
    for it in its[2:]:
        n, t = ob.roots_for_iteration(it)
        for r in ob.generate(n, t, it):
            sampled += int(r["sel_mask"].sum())
    dt = time.perf_counter() - t0
    return {"value": round(sampled / dt, 1), "unit": value_unit, "cores": int(ofinder.max_threads()),
            "kind": "port",
            "sample": (f"{sspec.name}: V={sspec.V} E={sspec.E} d_e={sspec.d_e} (events x{frac:g} of the GPU workload), "
                       f"{nb} batches of {spec.batch} spread over the epoch, f64 buffers like the reference "
                       f"(precision float64), numba prange + numpy on all cores; {cpu_model()}"),
            "ms_per_batch": round(dt / nb * 1e3, 2), "sample_build_s": round(build_s, 1)}


def import_reference():
    """tgadapt from baseline/_ref (the unmodified reference, pip-installed
    there by DESIGN.md's recipe), or None when it is absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "tgadapt")):
        return None
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tg_bench_numba")
    sys.path.insert(0, path)
    import tgadapt
    return tgadapt


def reference_graph(tg, spec, seed, its_fn):
    """The workload's graph in the reference's own types: events from the
    host twin of the device generator (oracle/shapes.py), T-CSR by the
    reference's build_graph.  Edge rows: the GDELT table is 142 GB, so it is
    a lazily committed host array (np.zeros) whose rows touched by the run's
    batches are written with their generator values before timing -- every
    row the reference reads holds its real value in real memory; rows it
    never reads are never committed."""
    import numpy as np
    from oracle import shapes as oshapes
    t0 = time.time()
    src, dst, ts = oshapes.synth_events(spec.V, spec.E, seed)
    eseed, nseed = oshapes.feature_seeds(seed)
    nf = oshapes.synth_features(0, spec.V, spec.d_v, nseed) if spec.d_v else None
    g = tg.build_graph(src, dst, ts, num_nodes=spec.V, node_features=nf)
    del src, dst, ts
    build_s = time.time() - t0
    if spec.d_e:
        g.edge_features = np.zeros((spec.E, spec.d_e), dtype=np.float32)
    return g, build_s, eseed


def reference_step(tg, trainer, it):
    """One mini-batch through the reference's own Trainer methods: the roots
    of train_iteration (training.py:375-382), _layer_neighborhoods per layer
    with hop expansion (_forward, training.py:301-314), and the PP phase's
    feature slices (training.py:318-321 graphmixer, :333-339 tgat) -- the
    aggregator math itself is not part of mini-batch generation.
    Returns (sampled neighbors, per-layer records)."""
    import numpy as np
    g, cfg = trainer.graph, trainer.cfg
    trainer.iteration = it
    eids = trainer._select_batch_eids(it)
    b = eids.size
    rng = tg.training.substream(trainer.seed, tg.training._S_NEG, it)
    negs = trainer.dst_pool[rng.integers(0, trainer.dst_pool.size, size=b)]
    nodes = np.concatenate([g.src[eids], g.dst[eids], negs])
    times = np.concatenate([g.ts[eids]] * 3)
    act = {trainer.L: (nodes, times)}
    recs = {}
    for l in range(trainer.L, 0, -1):
        tn, tt = act[l]
        rec = trainer._layer_neighborhoods(tn, tt, l, True, it)
        recs[l] = rec
        if l > 1:
            w = rec["sel_ids"].shape[1]
            act[l - 1] = (np.concatenate([tn, rec["sel_ids"].ravel()]),
                          np.concatenate([tt, np.repeat(tt, w) - rec["sel_dts"].ravel()]))
    t0 = time.perf_counter()
    if cfg.aggregator == "graphmixer":
        rec = recs[1]
        trainer._edge_feature_rows(rec["sel_eids"], rec["sel_mask"], True)
        trainer._node_feature_rows(rec["sel_ids"], rec["sel_mask"])
    else:
        for l in range(1, trainer.L + 1):
            rec = recs[l]
            trainer._edge_feature_rows(rec["sel_eids"], rec["sel_mask"], True)
            if l == 1:
                trainer._node_feature_rows(rec["sel_ids"], rec["sel_mask"])
                trainer._node_feature_rows(act[1][0])
    trainer.phase_seconds["PP"] += time.perf_counter() - t0
    return sum(int(r["sel_mask"].sum()) for r in recs.values()), recs


def run_reference(args, rank, world):
    if rank != 0:
        return
    spec = load_specs()[args.workload]
    tg = import_reference()
    if tg is None:
        return run_reference_port(args, spec, world)
    import numpy as np
    from oracle import shapes as oshapes
    t_all = time.time()
    steps = min(args.steps, REF_MAX_STEPS[spec.key])
    S = args.warmup + steps
    g, build_s, eseed = reference_graph(tg, spec, args.seed, None)
    cfg = tg.RunConfig(**{k: v for k, v in spec.config_fields().items() if k != "precision"},
                       adaptive_minibatch=False, precision="float32")
    split = tg.chronological_split(g, cfg.split_ratios)
    trainer = tg.Trainer(g, split, cfg, seed=0)
    its = step_iterations(S, 1, 0, trainer.iters_per_epoch)
    # untimed pass: which edge rows does the run read?  (fills them, see reference_graph)
    t0 = time.time()
    if spec.d_e and spec.E * spec.d_e * 4 <= FULL_FILL_BYTES:
        fill_rows(g.edge_features, None, spec.d_e, eseed)
    elif spec.d_e:
        touched = []
        read_rows = trainer._edge_feature_rows

        def record_rows(eids, mask, train_mode):  # instance-level hook, this pass only
            touched.append(eids[mask])
            return read_rows(eids, mask, train_mode)

        trainer._edge_feature_rows = record_rows
        for it in its:
            reference_step(tg, trainer, it)
        rows = np.unique(np.concatenate(touched))
        fill_rows(g.edge_features, rows, spec.d_e, eseed)
        trainer = tg.Trainer(g, split, cfg, seed=0)  # fresh cache counters / phase timers
    fill_s = time.time() - t0
    for s in range(args.warmup):
        reference_step(tg, trainer, its[s])
    for k in trainer.phase_seconds:
        trainer.phase_seconds[k] = 0.0
    sampled = 0
    t0 = time.perf_counter()
    for s in range(args.warmup, S):
        sampled += reference_step(tg, trainer, its[s])[0]
    dt = time.perf_counter() - t0
    value = sampled / dt
    import numba
    cores = int(numba.get_num_threads())
    sample = (f"full workload graph ({spec.E} events, reference build_graph T-CSR); {steps} timed batches of "
              f"{spec.batch} spread over the epoch (the same iterations as our arm), after {args.warmup} warm-up; "
              f"reference Trainer._layer_neighborhoods + hop expansion + _edge_feature_rows/_node_feature_rows, "
              f"precision float32 (f32 rows like ours), train mode with the cache; numba {cores} threads; "
              f"{cpu_model()}")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": "sampled neighbors/s",
           "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt / steps * 1e3, 3),
           "minibatch_gen_ms": round(dt / steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": DTYPE, "data": DATA, "config": workload_config(spec),
           "parallelism": f"host CPU, rank 0 only ({cores} numba threads)",
           "phase_seconds": {k: round(v, 4) for k, v in trainer.phase_seconds.items()},
           "cpu_baseline": {"value": round(value, 1), "unit": "sampled neighbors/s", "cores": cores,
                            "kind": "reference", "sample": sample},
           "e2e": {"value": round(value, 1), "unit": "sampled neighbors/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "setup_s": {"graph_build": round(build_s, 1), "row_fill": round(fill_s, 1),
                       "total": round(time.time() - t_all, 1)},
           "product_lib_mapped": product_lib_mapped()}
    print(json.dumps(out), flush=True)


FULL_FILL_BYTES = 40e9  # edge tables up to this size are written in full


def fill_rows(table, rows, d, seed, chunk=1 << 16):
    """table[rows] = generator rows (rows None: every row), on a thread pool
    (numpy releases the GIL in its loops)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import shapes as oshapes
    n = table.shape[0] if rows is None else rows.shape[0]

    def part(c0):
        if rows is None:
            table[c0:c0 + chunk] = oshapes.synth_features(c0, min(chunk, n - c0), d, seed)
        else:
            r = rows[c0:c0 + chunk]
            table[r] = oshapes.synth_feature_rows(r, d, seed)

    with ThreadPoolExecutor(os.cpu_count() or 1) as pool:
        list(pool.map(part, range(0, n, chunk)))


def product_lib_mapped():
    """True if this process has libtaser_b200.so mapped (it must not, here)."""
    try:
        with open("/proc/self/maps") as fh:
            return "libtaser_b200" in fh.read()
    except OSError:
        return None


def run_reference_port(args, spec, world):
    """No baseline/_ref: the oracle port (pinned to the reference's goldens)
    on a bounded event sample, labelled as such."""
    nb = max(1, args.steps) if args.cpu_batches is None else args.cpu_batches
    nb = min(nb, CPU_BATCHES[spec.key] * 2)
    args.cpu_batches = nb
    cb = cpu_baseline(args, spec, value_unit="sampled neighbors/s")
    cfg = workload_config(spec)
    out = {"impl": "reference", "metric": METRIC,
           "value": cb["value"], "unit": "sampled neighbors/s", "n_gpus": world, "steps": nb, "warmup": 2,
           "ms_per_step": cb["ms_per_batch"], "minibatch_gen_ms": cb["ms_per_batch"], "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": DTYPE, "data": DATA, "config": cfg,
           "timed_sample": cb["sample"],
           "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
           "e2e": {"value": cb["value"], "unit": "sampled neighbors/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks on 127.0.0.1 (one
    per GPU) with torch.distributed.run and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # init lines show nranks per communicator
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    rank, local_rank, world = dist_env()
    if world > 1 and args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
