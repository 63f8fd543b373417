"""Key ncu metrics per kernel: python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "Issue Slots Busy", "Executed Instructions", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "DRAM Throughput", "Compute (SM) Throughput",
        "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Block Limit Registers", "Block Limit Shared Mem", "Eligible Warps Per Scheduler",
        "No Eligible")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
seen = set()
for r in rows[1:]:
    key = (r[ii], r[mi])
    if r[mi] in WANT and key not in seen:
        seen.add(key)
        print(f"{r[ii]:>3} {r[ki][:34]:34s} {r[mi]:38s} {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
    if name in h:
        i = h.index(name)
        print(name, [r[i] for r in rows[2:]], rows[1][i])
