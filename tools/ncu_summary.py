"""Summarise an ncu report: time, DRAM traffic, stall reasons, hot source lines.

usage: python tools/ncu_summary.py report.ncu-rep [n_lines]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
          "launch__block_size", "launch__registers_per_thread",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"):
    if k in get:
        print(f"{k:60s} {get[k][0]} {get[k][1]}")
stalls = []
for h, (v, u) in get.items():
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in stalls) or 1
print("stall reasons (sampled):")
for x, h in sorted(stalls, reverse=True)[:8]:
    print(f"  {h:30s} {100 * x / tot:5.1f}%")
# hot CUDA source lines (cuda,sass view: per-line aggregate rows have Address "-")
txt = ncu("--page", "source", "--csv", "--print-source", "cuda,sass")
agg = []
fname = "?"
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[2] == "-" and r[0].isdigit():
        try:
            agg.append((int(r[4]), f"{fname}:{r[0]}", r[1].strip()[:100]))
        except ValueError:
            pass
t2 = sum(a for a, _, _ in agg) or 1
print("hot source lines (stall samples):")
for a, l, s in sorted(agg, reverse=True)[:top]:
    print(f"  {100 * a / t2:5.1f}%  {l}: {s}")
