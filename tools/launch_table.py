"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        h, start = r, i
        break
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = defaultdict(list)
for r in rows[start + 1:]:
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0) * v
    d[r[ki].split("(")[0][-48:]].append(v)
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:48s} n={len(v):4d} mean_us={sum(v)/len(v):9.1f} total_us={sum(v):10.1f} {100*sum(v)/tot:5.1f}%")
