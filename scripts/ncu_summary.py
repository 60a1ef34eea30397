"""Summarise an ncu report (--page raw) or a launch list CSV into markdown.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep  > profiles/rNN_x.md
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__waves_per_multiprocessor", "waves/SM"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long-scoreboard/issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg-throttle/issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier/issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math-throttle/issue"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"ncu --set full summary of `{path}`\n")
    for n, r in enumerate(rows[2:]):
        d = dict(zip(hdr, r))
        print(f"### launch {n}: `{d.get('Kernel Name')}` grid {d.get('Grid Size')} block {d.get('Block Size')}\n")
        print("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in d:
                print(f"| {label} (`{key}`) | {d[key]} {units[hdr.index(key)]} |")
        print()


def launches(path):
    text = open(path).read().splitlines()
    i = next(k for k, line in enumerate(text) if line.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[i:]))))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = (r["Kernel Name"].split("(")[0], r["Grid Size"])
        v = float(r["Metric Value"]) / (1e3 if r["Metric Unit"] == "ns" else 1.0)
        agg[k][0] += 1
        agg[k][1] += v
        total += v
    print(f"launch list `{path}` ({sum(a[0] for a in agg.values())} launches, {total:.1f} us total)\n")
    print("| kernel | grid | launches | total us | mean us | share |\n|---|---|---|---|---|---|")
    for (name, grid), (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {grid} | {n} | {us:.1f} | {us / n:.1f} | {us / total:.1%} |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        report(sys.argv[1])
