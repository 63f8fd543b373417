"""Print the hottest SASS instructions (by executed warp instructions) of each
kernel in an ncu report: python tools/sass_hot.py report.ncu-rep [kernel-substr] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    lines = b.split("\n")
    kname = lines[0]
    if want not in kname:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ie = h.index("Instructions Executed")
    src = h.index("Source")
    st = h.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ie] or 0), int(r[st] or 0), i, r[src].strip()) for i, r in enumerate(rows[1:]) if len(r) > ie]
    tot = sum(d[0] for d in data)
    tots = sum(d[1] for d in data)
    print(f"== {kname[:90]}  total warp-instr {tot:.3e}  stall samples {tots}")
    # print in address order the instructions with >= 0.3% of executions, plus hottest stalls
    for n, s, i, text in data:
        if n >= 0.003 * tot or s >= 0.01 * tots:
            print(f"{i:5d} {n/tot*100:6.2f}% st{s/tots*100:5.1f}%  {text}")
