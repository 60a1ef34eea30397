"""Overlap summary of a bench.py --trace kernel timeline (JSON lines):
per-kernel busy time, time with 0/1/2/3+ kernels active, and the share of
the span in which a row-gather kernel is running."""
import collections
import json
import sys

ev = [json.loads(line) for line in open(sys.argv[1])]
span0, span1 = min(e["start"] for e in ev), max(e["end"] for e in ev)
by = collections.defaultdict(lambda: [0, 0.0])
pts = []
for e in ev:
    by[e["name"][:60]][0] += 1
    by[e["name"][:60]][1] += e["end"] - e["start"]
    g = "gather" in e["name"]
    pts += [(e["start"], 1, g), (e["end"], -1, g)]
pts.sort()
active = gact = 0
last = span0
hist = collections.Counter()
gtime = 0.0
for t, d, g in pts:
    hist[min(active, 3)] += t - last
    if gact > 0:
        gtime += t - last
    last = t
    active += d
    gact += d if g else 0
span = span1 - span0
print(f"span {span:.1f} us, {len(ev)} kernels")
for k, (n, t) in sorted(by.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us {n:4d}x  {k}")
print("concurrency share:", {k: round(v / span, 3) for k, v in sorted(hist.items())})
print(f"row gather active {gtime / span:.3f} of the span")
