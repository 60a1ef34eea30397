"""Per-kernel time and DRAM bytes of an ncu --csv launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum:
python scripts/launch_bw.py launches.csv [regex]"""
import collections
import csv
import re
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = [r for r in csv.reader(open(sys.argv[1]))]
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
per = collections.OrderedDict()
for d in data:
    key = (d["ID"], d["Kernel Name"])
    v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", ""), 1.0)
    per.setdefault(key, {})[d["Metric Name"]] = v
agg = collections.OrderedDict()
for (i, name), m in per.items():
    short = name.split("(")[0][:70]
    if pat and not pat.search(name):
        continue
    a = agg.setdefault(short, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
print(f"{'kernel':70s} {'n':>4s} {'us':>10s} {'DRAM MB':>10s} {'GB/s':>8s}")
for k, (n, us, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} {n:4d} {us:10.1f} {(rd + wr) / 1e6:10.1f} {(rd + wr) / max(us, 1e-9) / 1e3:8.1f}")
