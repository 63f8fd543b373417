"""Executed instructions and stall samples of one kernel per CUDA source line:
joins an ncu report's SASS page (per-instruction counts, by address) with the
line table of the same build's cubin (nvdisasm -g, by function offset).

python tools/ncu_lines.py report.ncu-rep file.cubin kernel-substr [min-share]
"""
import csv
import io
import re
import subprocess
import sys

rep, cubin, want = sys.argv[1], sys.argv[2], sys.argv[3]
min_share = float(sys.argv[4]) if len(sys.argv) > 4 else 0.005

# per-offset source line of the kernel in the cubin
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
fn, cur, lines = None, None, {}
for line in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        fn = m.group(1)
        continue
    if fn is None or want not in fn:
        continue
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)', line)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
    if fn and want in fn and lines and re.match(r"\s*\.text\.", line):
        break

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
blocks = out.split('"Kernel Name"')
agg, tot_i, tot_s = {}, 0, 0
for b in blocks[1:]:
    rows = b.split("\n")
    if want.split("I")[0].replace("_Z", "") not in rows[0] and want not in rows[0]:
        pass
    data = list(csv.reader(io.StringIO("\n".join(rows[1:]))))
    h = data[0]
    if "Instructions Executed" not in h:
        continue
    ai, ie, st = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in data[1:] if len(r) > ie]
    if not body:
        continue
    base = int(body[0][ai], 16)
    if len(body) != len(lines) and abs(len(body) - len(lines)) > 8:
        continue  # another kernel
    for r in body:
        off = int(r[ai], 16) - base
        key = lines.get(off, "?")
        i, s = int(r[ie] or 0), int(r[st] or 0)
        a = agg.setdefault(key, [0, 0])
        a[0] += i
        a[1] += s
        tot_i += i
        tot_s += s
    break
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][0]):
    if i / max(tot_i, 1) >= min_share or s / max(tot_s, 1) >= min_share:
        print(f"{k:28s} instr {100 * i / tot_i:5.1f}%  stall {100 * s / max(tot_s, 1):5.1f}%")
print(f"total executed {tot_i}")
