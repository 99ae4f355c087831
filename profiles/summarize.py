"""Summarise ncu outputs into profiles/ (committed evidence).

    python profiles/summarize.py launches <launches.csv>      # per-kernel share of a bench step
    python profiles/summarize.py details <report.ncu-rep>     # key metrics per profiled kernel
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "No Eligible", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) > vi:
            agg[r[ki][:100]][0] += 1
            agg[r[ki][:100]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"{'total ms':>10} {'n':>4} {'share':>6}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v[1] / 1e6:10.3f} {v[0]:4d} {100 * v[1] / tot:5.1f}%  {k}")


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mn, mu, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    cur = None
    for r in rows[1:]:
        if r[ki] != cur:
            cur = r[ki]
            print(f"== {cur[:110]}")
        if r[mn] in KEYS:
            print(f"   {r[mn]:40s} {r[mv]} {r[mu]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if rr:
        h = rr[0]
        want = [i for i, n in enumerate(h) if n in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                                     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                                                     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                                                     "gpu__time_duration.sum")]
        print("\nraw:")
        print(" | ".join(h[i] for i in want))
        for r in rr[2:]:
            print(" | ".join(r[i][:60] for i in want))


if __name__ == "__main__":
    {"launches": launches, "details": details}[sys.argv[1]](sys.argv[2])
