"""Executed-instruction mix by opcode of one kernel in an ncu report:
python tools/ncu_opmix.py report.ncu-rep kernel-substr"""
import csv
import io
import re
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
for b in out.split('"Kernel Name"')[1:]:
    lines = b.split("\n")
    if want not in lines[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    si, ie = h.index("Source"), h.index("Instructions Executed")
    agg, tot = {}, 0
    for r in rows[1:]:
        if len(r) <= ie:
            continue
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", r[si])
        if not m:
            continue
        n = int(r[ie] or 0)
        agg[m.group(1)] = agg.get(m.group(1), 0) + n
        tot += n
    for k, v in sorted(agg.items(), key=lambda x: -x[1])[:30]:
        print(f"{k:10s} {100 * v / tot:5.1f}%")
    print("total", tot)
    break
