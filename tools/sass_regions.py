"""Aggregate executed instructions and stall samples of one kernel's SASS by
address region, printing region boundaries' instructions so phases can be
identified: python tools/sass_regions.py report.ncu-rep kernel-substr [lines-per-region]"""
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
step = int(sys.argv[3]) if len(sys.argv) > 3 else 100
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
for b in out.split('"Kernel Name"')[1:]:
    lines = b.split("\n")
    if want not in lines[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ie] or 0), int(r[st] or 0), r[src].strip()) for r in rows[1:] if len(r) > ie]
    tot, tots = sum(d[0] for d in data), sum(d[1] for d in data)
    for a in range(0, len(data), step):
        chunk = data[a:a + step]
        ni, ns = sum(c[0] for c in chunk), sum(c[1] for c in chunk)
        marks = [c[2] for c in chunk if any(k in c[2] for k in ("BAR", "MATCH", "ATOMG", "RED", "CCTL", "EXIT"))][:4]
        print(f"{a:5d}-{a + len(chunk) - 1:5d} instr {100 * ni / max(tot, 1):6.2f}% stall {100 * ns / max(tots, 1):6.2f}%  {' | '.join(m[:40] for m in marks)}")
    break
