"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_summary.py launches.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 10
hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * {"usecond": 1e3, "msecond": 1e6}.get(r[ui], 1.0)
    k = r[ki][:70]
    tot[k] += v
    cnt[k] += 1
T = sum(tot.values()) or 1.0
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / T:5.1f}%  {cnt[k]:4d} x {v / cnt[k] / 1e6:8.3f} ms  {k}")
