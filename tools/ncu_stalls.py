"""Per-kernel issue/stall/pipe summary of an ncu --set full report:
python tools/ncu_stalls.py report.ncu-rep [kernel-regex] > summary.txt

For every profiled launch: duration, executed warp-instructions, issue-slot
and occupancy figures, the stall breakdown (cycles per issued instruction,
smsp__average_warps_issue_stalled_*_per_issue_active) and the pipe
utilisations (sm__inst_executed_pipe_*, % of peak while active)."""

import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, rows = rows[0], rows[2:]
col = {c: i for i, c in enumerate(h)}


def g(row, name, default=float("nan")):
    i = col.get(name)
    if i is None or row[i] in ("", "n/a"):
        return default
    try:
        return float(row[i].replace(",", ""))
    except ValueError:
        return row[i]


STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$")
PIPE = re.compile(r"sm__inst_executed_pipe_(\w+)\.avg\.pct_of_peak_sustained_active$")
for row in rows:
    name = row[col["Kernel Name"]]
    if pat and not pat.search(name):
        continue
    short = name.split("(")[0]
    print(f"== {short}  grid {row[col['launch__grid_size']]} x {row[col['launch__block_size']]}, "
          f"{row[col['launch__registers_per_thread']]} regs")
    print(f"   duration {g(row, 'gpu__time_duration.sum'):.2f} us, "
          f"warp-instr {g(row, 'smsp__inst_executed.sum') / 1e6:.2f} M, "
          f"issue active {g(row, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} %, "
          f"warps active {g(row, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} % "
          f"(theoretical {g(row, 'sm__maximum_warps_per_active_cycle_pct'):.1f} %), "
          f"eligible/scheduler {g(row, 'smsp__warps_eligible.avg.per_cycle_active'):.2f}, "
          f"DRAM {g(row, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} %")
    stalls = sorted(((float(row[i] or 0), m.group(1)) for c, i in col.items()
                     if (m := STALL.match(c)) and row[i] not in ("", "n/a")), reverse=True)
    tot = sum(v for v, _ in stalls)
    print("   stalls (cycles/issue, total %.2f): " % tot +
          ", ".join(f"{k} {v:.2f}" for v, k in stalls if v >= 0.05))
    pipes = sorted(((float(row[i] or 0), m.group(1)) for c, i in col.items()
                    if (m := PIPE.match(c)) and row[i] not in ("", "n/a")), reverse=True)
    print("   pipes (% active): " + ", ".join(f"{k} {v:.1f}" for v, k in pipes if v >= 1.0))
