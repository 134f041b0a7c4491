"""ptxas -v summary: kernel, registers, spill bytes.  usage: nvcc ... -Xptxas -v 2>&1 | python ptxas_regs.py [filter]"""
import re, sys
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1); rows[cur] = [None, None]; continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur: rows[cur][1] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur: rows[cur][0] = int(m.group(1))
for k, (r, sp) in sorted(rows.items()):
    if flt in k:
        print(f"{k[:70]:70s} regs={r} spill={sp}")
