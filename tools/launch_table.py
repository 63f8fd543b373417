"""Print the last frame's kernels from an ncu --metrics gpu__time_duration.sum
--csv launch list: python tools/launch_table.py launches.csv [frames]"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h, rows = rows[0], rows[1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 2
tot = 0.0
for r in rows[len(rows) - len(rows) // frames:]:
    us = float(r[vi].replace(",", "")) / 1000
    tot += us
    print(f"{us:8.1f} us  {r[ki][:90]}")
print(f"{tot:8.1f} us  total")
