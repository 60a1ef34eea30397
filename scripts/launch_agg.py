"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"])
    unit = d.get("Metric Unit", "")
    v = v / 1000 if unit in ("nsecond", "ns") else (v * 1000 if unit == "msecond" else v)
    a = agg.setdefault(d["Kernel Name"][:70], [0, 0.0])
    a[0] += 1
    a[1] += v
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t:10.1f} us {n:5d}x {k}")
