"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per
(kernel, grid): launches, mean and total duration, share of the total.

  python tools/launch_shares.py gpurun_out/launches_bench.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ki, gi, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Grid Size", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        key = (r[ki].split("(")[0][:64], r[gi])
        agg[key][0] += 1
        agg[key][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(v[1] for v in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"{'share':>6} {'launches':>8} {'mean us':>10} {'total ms':>9}  kernel [grid]")
for (k, g), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{100 * t / tot:5.1f}% {n:8d} {t / n:10.1f} {t / 1e3:9.2f}  {k} {g}")
