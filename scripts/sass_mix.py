"""Instruction mix + stall samples of an `ncu --page source --csv --print-source sass` export
(optionally per source-line range): python scripts/sass_mix.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
tot = sum(int(d["Instructions Executed"] or 0) for d in data)
samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total warp instr", tot, "stall samples", samp)
op, st = collections.Counter(), collections.Counter()
for d in data:
    m = d["Source"].split()
    o = m[1] if m[0].startswith("@") else m[0]
    op[o] += int(d["Instructions Executed"] or 0)
    st[o] += int(d["Warp Stall Sampling (All Samples)"] or 0)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for o, c in op.most_common(top):
    print(f"{o:34s} {c:12d} {c / max(tot, 1):.3f} stall_samples {st[o]}")
print("-- hottest instructions by stall samples")
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:25]:
    print(d["Address"][-5:], f"{int(d['Warp Stall Sampling (All Samples)'] or 0):6d}", f"{int(d['Instructions Executed'] or 0):10d}", d["Source"][:90])
