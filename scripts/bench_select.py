"""K9 microbenchmark: importance-weighted batch selection at the GDELT
training-split size.

    python scripts/bench_select.py [--n 114774529] [--b 600] [--iters 20]

Times tg_select_batch (CUDA events, scores resident in HBM) against the
reference algorithm on the host (oracle.selector.select_batch == numpy's
Generator.choice, single-threaded like the reference), same scores and
streams, and checks the device result equals the host one.  Prints one JSON
line.  Algorithmic bytes per selection (one choice() round, the case when
b << n): the scores are read once for numpy's pairwise total and once for
the exact sequential cumsum of p = scores/total (p is never materialised):
16 B per training edge.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=int(0.6 * 191_290_882))
    ap.add_argument("--b", type=int, default=600)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cpu-iters", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch
    from oracle import selector as osel
    from paper_2402_05396_b200 import selector as dsel
    from paper_2402_05396_b200.seeds import S_BATCH, substream

    host = 1.0 / (1.0 + np.exp(-np.random.default_rng(0).normal(size=args.n) * 3)) + 0.1
    sc = dsel.as_scores(host, 0.1)
    for it in range(2):  # warm-up + parity
        got = dsel.select_batch(sc, args.b, substream(0, S_BATCH, it)).cpu().numpy()
        exp = osel.select_batch(host, args.b, substream(0, S_BATCH, it))
        assert np.array_equal(got, exp), "device selection differs from numpy"
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(args.iters):
        dsel.select_batch(sc, args.b, substream(0, S_BATCH, 100 + it))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.iters
    t0 = time.perf_counter()
    for it in range(args.cpu_iters):
        osel.select_batch(host, args.b, substream(0, S_BATCH, 200 + it))
    cpu_ms = (time.perf_counter() - t0) / args.cpu_iters * 1e3
    algo = args.n * 16
    peak = 6553.3
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except Exception:
        pass
    gbs = algo / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": "K9 tg_select_batch", "n": args.n, "b": args.b, "ms_per_selection": round(ms, 4),
                      "algorithmic_bytes": algo, "GB/s": round(gbs, 1), "hbm_frac": round(gbs / peak, 4),
                      "cpu_reference_ms": round(cpu_ms, 1), "cpu_kind": "numpy Generator.choice (single thread)",
                      "speedup": round(cpu_ms / ms, 1), "bit_exact": True}))


if __name__ == "__main__":
    main()
