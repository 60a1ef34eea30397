"""Print the kernel sequence of the last step in an ncu launch-list CSV."""
import csv
import io
import sys

text = open(sys.argv[1]).read().splitlines()
first = sys.argv[2] if len(sys.argv) > 2 else "find_kernel"
i = next(k for k, line in enumerate(text) if line.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(text[i:]))))
names = [(r["Kernel Name"].split("(")[0][:60], float(r["Metric Value"]) / 1e3) for r in rows
         if r["Metric Name"] == "gpu__time_duration.sum"]
idx = [k for k, (n, _) in enumerate(names) if first in n]
tot = 0.0
for n, us in names[idx[-1]:]:
    print(f"{us:9.1f} us  {n}")
    tot += us
print(f"total {tot:.1f} us")
