"""One launch each of the once-per-graph / once-per-epoch / small kernels at
the benchmarked sizes, for single-kernel ncu captures:

  K1  tg_tcsr_build at GDELT scale (191,290,882 events, 382.6M entries)
  K6  tg_cache_replace at k = 0.2 E = 38.26M over E int32 counters
  K8  tg_sample_wor at the MovieLens shape (B = 12,000, m = 25, n = 10)

    ncu --set full --clock-control none -k regex:'<kernels>' python scripts/evidence_kernels.py

Prints the CUDA-event time of each call (not under a profiler, these are the
numbers to quote)."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    from paper_2402_05396_b200 import build_graph, make_cache, maybe_replace
    from paper_2402_05396_b200.sampler import sample_wor_device
    from paper_2402_05396_b200.shapes import synth_events_device
    from paper_2402_05396_b200.specs import SHAPES
    which = sys.argv[1:] or ["k1", "k6", "k8"]
    spec = SHAPES["E"]
    torch.cuda.set_device(0)
    if "k1" in which:
        src, dst, ts = synth_events_device(spec.V, spec.E, 0)
        g, ms = timed(lambda: build_graph(src, dst, ts, num_nodes=spec.V))
        print(f"K1 build_graph E={spec.E}: {ms:.1f} ms ({2 * spec.E} entries)", flush=True)
        del g, src, dst, ts
        torch.cuda.empty_cache()
    if "k6" in which:
        E = spec.E
        cache = make_cache(E, 0.2)
        gen = torch.Generator(device="cuda").manual_seed(1)
        # an epoch's access counts: 60% of the edges touched, heavy-tailed
        touched = torch.rand(E, device="cuda", generator=gen) < 0.6
        cnt = torch.floor(torch.rand(E, device="cuda", generator=gen).pow(-0.7)).to(torch.int32)
        cache.counters_i32.copy_(torch.where(touched, cnt, torch.zeros_like(cnt)))
        for epoch in range(2):
            _, ms = timed(lambda: maybe_replace(cache))
            print(f"K6 maybe_replace E={E} k={cache.k} epoch {epoch}: {ms:.1f} ms", flush=True)
            cache.counters_i32.copy_(torch.where(touched, cnt.roll(epoch + 1), torch.zeros_like(cnt)))
    if "k8" in which:
        B, m, n = 12000, 25, 10
        rng = np.random.default_rng(0)
        logits = rng.normal(size=(B, m))
        mask = rng.random((B, m)) < 0.9
        e = np.where(mask, np.exp(logits - logits.max(axis=1, keepdims=True)), 0.0)
        q = torch.as_tensor(e / np.maximum(e.sum(axis=1, keepdims=True), 1e-300)).cuda()
        lq = torch.log(q.clamp_min(1e-300))
        for it in range(3):
            _, ms = timed(lambda: sample_wor_device(q, lq, n, np.random.default_rng(it)))
            print(f"K8 sample_wor B={B} m={m} n={n}: {ms * 1e3:.1f} us", flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"done in {time.time() - t0:.1f} s")
