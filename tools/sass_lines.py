"""Static SASS census of one kernel by source line (needs -lineinfo):
python tools/sass_lines.py file.cubin kernel-substr [OPCODE_PREFIX ...]
Prints, per source line, the count of instructions whose opcode starts with
one of the prefixes (default: local-memory traffic STL/LDL), so spills on the
hot loop can be told apart from spills around rare calls."""
import re
import subprocess
import sys

cubin, want = sys.argv[1], sys.argv[2]
prefixes = tuple(sys.argv[3:]) or ("STL", "LDL")
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
fn = None
cur = None
stats = {}
total = {}
for line in out.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        fn = m.group(1)
        continue
    if fn is None or want not in fn:
        continue
    m = re.search(r'//## File "[^"]*/([^"/]+)", line (\d+)', line)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        op = m.group(1)
        total[cur] = total.get(cur, 0) + 1
        if op.startswith(prefixes):
            stats.setdefault(cur, []).append(op)
for k in sorted(stats):
    print(f"{k[0]}:{k[1]}  {len(stats[k])}/{total[k]}  {' '.join(stats[k][:8])}")
