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
    p.add_argument("--inflight", type=int, default=3, help="mini-batches in flight (generator slots)")
    p.add_argument("--placement", default="auto", choices=["auto", "replicated", "sharded"],
                   help="edge-feature placement (placement.py): auto = replicated when the table fits one GPU")
    return p.parse_args()


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

    def _run(self):
        while not self._stop.is_set():
            if self.nv is not None:
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    for name, bit in self._NAMES.items():
                        if r & bit:
                            self.reasons.add(name)
                except Exception:
                    pass
            time.sleep(0.001)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

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
    # multi-rank timing / reduction logic on a 1-GPU box; NCCL forbids two
    # ranks on one device).  Normal runs: one rank per GPU over NCCL.
    share = os.environ.get("TG_BENCH_SHARE_GPU") == "1"
    dev_index = 0 if share else local_rank
    torch.cuda.set_device(dev_index)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    red_dev = "cpu" if share else "cuda"
    from paper_2402_05396_b200 import _lib
    from paper_2402_05396_b200.pipeline import MiniBatchGenerator
    from paper_2402_05396_b200.shapes import SHAPES, make_graph

    spec = SHAPES[args.workload]
    placement = args.placement
    if placement == "auto":
        # replicate when table + T-CSR + cache state fit in 90% of this GPU's HBM
        need = spec.E * (4 * ((spec.d_e + 3) & ~3) + 2 * 16 + 8 + 24) + spec.V * 8
        total = torch.cuda.get_device_properties(dev_index).total_memory
        placement = "replicated" if need * (2 if share else 1) < 0.9 * total else "sharded"
    t0 = time.time()
    g = make_graph(spec, seed=args.seed, edge_placement=placement)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    cfg = spec.path_config()
    gen = MiniBatchGenerator(g, cfg, seed=0)
    S = args.warmup + args.steps
    iters = gen.iters_per_epoch
    # batch index of step s on this rank: spread over the epoch, ranks interleaved
    its = [((s * world + rank) * iters) // (S * world) for s in range(S)]
    roots = []
    for it in its:
        n, tt = gen.roots_for_iteration(it)
        roots.append((torch.as_tensor(n).cuda(), torch.as_tensor(tt).cuda()))
    seeds = [gen.seeds_for(it) for it in its]
    stream = torch.cuda.current_stream()

    K = max(1, args.inflight)

    def step(s, events=None, slot=0):
        return gen.generate(roots[s][0], roots[s][1], its[s], finder_seeds=seeds[s], events=events, slot=slot)

    # the previous epoch (same positive edges, other negatives: it + iters)
    # counts accesses; its epoch boundary fills the cache (cache.py:107-118),
    # so the timed steps see the reference's steady-state resident set --
    # with sharded placement, the replicated hot tier
    if gen.cache is not None:
        for s in range(S):
            pn, pt = gen.roots_for_iteration(its[s] + iters)
            gen.generate(torch.as_tensor(pn).cuda(), torch.as_tensor(pt).cuda(), its[s] + iters)
        if world > 1:
            from paper_2402_05396_b200.shard import epoch_allreduce
            torch.cuda.synchronize()
            cnt = gen.cache.counters_i32 if not share else gen.cache.counters_i32.cpu()
            epoch_allreduce([cnt])
            if share:
                gen.cache.counters_i32.copy_(cnt)
        gen.end_epoch()
        gen.cache.stats.zero_()

    # accounting pass: algorithmic bytes + sampled neighbors of every step (untimed)
    acct = []
    for s in range(S):
        recs = step(s)
        per = [layer_bytes(g, r, g.d_e, gen.cache is not None) for r in recs]
        for p_, r in zip(per, recs):
            p_["sampled"] = int(r["sel_mask"].sum().item())
        acct.append(per)
    torch.cuda.synchronize()

    # warm-up
    for s in range(args.warmup):
        step(s, slot=s % K)
    gen.join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # timed pass A: the step loop as a user runs it
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for k in range(1, K):
            gen.slot_stream(k).wait_stream(stream)
        for s in range(args.warmup, S):
            step(s, slot=s % K)
        gen.join(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
    sampled = sum(sum(p["sampled"] for p in acct[s]) for s in range(args.warmup, S))
    samp_t = torch.tensor([float(sampled)], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(samp_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    total_sampled = float(samp_t.item())
    value = total_sampled / (ms_max / 1e3)

    # timed pass A1: single-batch latency ("mini-batch gen ms"):
    # the same steps with ONE batch in flight, so no batch overlaps another
    torch.cuda.synchronize()
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
    roofline = {"bound": "hbm", "kernel": "tg::row_gather_bulk_kernel (K5 edge-row slice on the bulk-copy engine, dominant)",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4),
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else
                f"fallback {HBM_FALLBACK_GBS} GB/s (B200_PROFILING.md)",
                "traffic": traffic,
                "algorithmic_bytes_per_launch": round(gby / n_launch),
                "avg_launch_us": round(gms / n_launch * 1e3, 2),
                "finder": {"kernel": "tg::find_kernel (K2+K3)", "avg_launch_us": round(fms / n_launch * 1e3, 2),
                           "algorithmic_bytes_per_launch": round(fby / n_launch),
                           "GB/s": round(fby / (fms / 1e3) / 1e9, 1)},
                "path": {"bytes_per_step": round((gby + fby) / args.steps),
                         "GB/s_over_step": round((gby + fby) / (ms / 1e3) / 1e9, 1),
                         "frac_over_step": round((gby + fby) / (ms / 1e3) / 1e9 / peak, 4)},
                "per_layer": [{"layer": gen.L - li, "roots": acct[args.warmup][li]["B"],
                               "find_us": round(f_ms[li] / args.steps * 1e3, 2),
                               "gather_us": round(g_ms[li] / args.steps * 1e3, 2),
                               "gather_GB/s": round(g_by[li] / (g_ms[li] / 1e3) / 1e9, 1)} for li in range(L)],
                "share_of_step": round(gms / max(ms, 1e-9), 3)}

    if spec.adaptive:
        # adaptive workloads: the dominant kernel is K7 scoring (tensor-bound)
        model = gen._adaptive.model
        k7_ms = sum(sev[s][li][0].elapsed_time(sev[s][li][1]) for s in range(args.warmup, S) for li in range(L))
        k7_flops = sum(model.flops(acct[s][li]["B"]) for s in range(args.warmup, S) for li in range(L))
        bf16 = float(peaks.get("bf16_tflops", 1647.8))
        tf32_peak = 0.5 * bf16
        ach = k7_flops / (k7_ms / 1e3) / 1e12
        k7 = {"bound": "tensor", "kernel": "K7 tg_score: tcgen05 3xTF32 GEMMs (tc_gemm_kernel) + encoders, token "
                                           "mixer, decoder, masked softmax",
              "achieved": round(ach, 2), "peak": round(tf32_peak, 1), "unit": "TFLOP/s",
              "frac": round(ach / tf32_peak, 4), "traffic": None,
              "peak_source": "measured bf16_tflops x 0.5 (dense TF32 rate); achieved counts useful FLOPs -- the "
                             "3xTF32 split issues 3 tf32 MMAs per product, so 1/3 is the ceiling" if model.tensor_cores
                             else "FFMA path (trans decoder)",
              "precision": model.precision, "tensor_cores": model.tensor_cores,
              "avg_us_per_layer": round(k7_ms / (args.steps * L) * 1e3, 2),
              "flops_per_step": round(k7_flops / args.steps), "share_of_step": round(k7_ms / max(ms, 1e-9), 3),
              "hbm": {"scope": "whole step: all algorithmic bytes (finder, candidate + selected rows) / step time",
                      "achieved": roofline["path"]["GB/s_over_step"], "peak": peak, "unit": "GB/s",
                      "frac": roofline["path"]["frac_over_step"]}}
        roofline = k7

    hit_rate = None
    if gen.cache is not None:
        hm = gen.cache.stats.cpu().tolist()
        hit_rate = round(hm[0] / max(1, hm[0] + hm[1]), 4)

    # end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, gen, its, seeds, acct, world, dist, red_dev)

    result = {
        "metric": METRIC,
        "value": round(value, 1), "unit": "sampled neighbors/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 ts / int64 ids / f32 rows",
        "data": "synthetic (device shape generator, SURVEY §8(d)); random-hash f32 features",
        "config": {"workload": f"{spec.key}:{spec.name}-shaped V={spec.V} E={spec.E} d_e={spec.d_e} d_v={spec.d_v}",
                   "path": spec.note, "batch": spec.batch, "roots_per_step": 3 * spec.batch,
                   "aggregator": spec.aggregator, "finder_policy": spec.finder_policy,
                   "adaptive": spec.adaptive, "cache_fraction": 0.2,
                   "parallelism": f"root-sharded weak scaling x{world} (replicated T-CSR, {placement} edge table)",
                   "edge_placement": placement, "cache_hit_rate": hit_rate,
                   "inflight": args.inflight,
                   "l2": "inputs larger than L2 (table + T-CSR >> 126 MB); batches spread over the epoch",
                   "graph_build_s": round(build_s, 2)},
        "sampled_per_step": round(total_sampled / world / args.steps, 1),
        "minibatch_gen_ms": round(gen_ms, 4),
        "minibatch_gen_ms_note": f"single-batch latency: device roots -> every buffer of the step ready, one batch in "
                                 f"flight (ms_per_step is the steady state with {K} in flight)",
        "gpu_launches": int(launches),
        "roofline": roofline,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(args, spec, value_unit="sampled neighbors/s")
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, gen, its, seeds, acct, world, dist, red_dev="cuda"):
    """The user's call with HOST buffers: pinned roots -> device, generate,
    every output of the step (ids/eids/dts/mask per layer + edge rows) back
    into pinned host memory, all inside the timed region.  With --inflight K
    the copies of batch i overlap the generation of batch i+1 (K slots, each
    with its own stream, device roots and pinned output buffers)."""
    import torch
    S = args.warmup + args.steps
    K = max(1, args.inflight)
    host_roots = []
    for it in its:
        n, t = gen.roots_for_iteration(it)
        host_roots.append((torch.as_tensor(n).pin_memory(), torch.as_tensor(t).pin_memory()))
    R1 = int(host_roots[0][0].shape[0])
    dv = [torch.empty(R1, dtype=torch.int64, device="cuda") for _ in range(K)]
    dt = [torch.empty(R1, dtype=torch.float64, device="cuda") for _ in range(K)]
    keys = ("sel_ids", "sel_eids", "sel_dts", "sel_mask", "edge_rows", "node_rows", "tgt_rows")
    recs = gen.generate(dv[0].copy_(host_roots[0][0]), dt[0].copy_(host_roots[0][1]), its[0], finder_seeds=seeds[0])
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
            out = gen.generate(dv[k], dt[k], its[s], finder_seeds=seeds[s], slot=k)
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
    samp_t = torch.tensor([float(samp)], device=red_dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(samp_t, op=dist.ReduceOp.SUM)
    return {"value": round(float(samp_t.item()) / (float(ms_t.item()) / 1e3), 1), "unit": "sampled neighbors/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(float(ms_t.item()) / args.steps, 4),
            "pcie_GB/s": round((h2d + d2h) / (float(ms_t.item()) / args.steps / 1e3) / 1e9, 1),
            "note": f"pinned host roots in, every mini-batch buffer (incl. f32 feature rows) out, per step; "
                    f"{K} batches in flight"}


# ---------------------------------------------------------------------------
# CPU reference (oracle port) on a bounded sample of the same workload
# ---------------------------------------------------------------------------

CPU_SAMPLE = {"A": 1.0, "B": 1.0, "C": 0.02, "D": 0.25, "E": 1 / 16}
CPU_BATCHES = {"A": 40, "B": 20, "C": 2, "D": 4, "E": 20}


def cpu_baseline(args, spec, value_unit):
    import numpy as np
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
    ob = OracleMiniBatch(og, sspec.path_config(), seed=0)
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
    cpu = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"value": round(sampled / dt, 1), "unit": value_unit, "cores": int(ofinder.max_threads()),
            "kind": "port",
            "sample": (f"{sspec.name}: V={sspec.V} E={sspec.E} d_e={sspec.d_e} (events x{frac:g} of the GPU workload), "
                       f"{nb} batches of {spec.batch} spread over the epoch, f64 buffers like the reference "
                       f"(precision float64), numba prange + numpy on all cores; {cpu}"),
            "ms_per_batch": round(dt / nb * 1e3, 2), "sample_build_s": round(build_s, 1)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2402_05396_b200.shapes import SHAPES
    spec = SHAPES[args.workload]
    nb = max(1, args.steps) if args.cpu_batches is None else args.cpu_batches
    nb = min(nb, CPU_BATCHES[spec.key] * 2)
    args.cpu_batches = nb
    cb = cpu_baseline(args, spec, value_unit="sampled neighbors/s")
    out = {"impl": "reference", "metric": METRIC,
           "value": cb["value"], "unit": "sampled neighbors/s", "n_gpus": world, "steps": nb, "warmup": 2,
           "ms_per_step": cb["ms_per_batch"], "minibatch_gen_ms": cb["ms_per_batch"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (host shape generator twin)",
           "config": {"workload": f"{spec.key}:{spec.name}-shaped V={spec.V} E={spec.E} d_e={spec.d_e}",
                      "path": spec.note},
           "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
           "e2e": {"value": cb["value"], "unit": "sampled neighbors/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
