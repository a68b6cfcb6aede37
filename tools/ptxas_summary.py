"""Summarise `nvcc -Xptxas -v` output: one line per kernel with registers / spills / smem."""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
rows = []
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = [r["name"] for r in rows]
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
except Exception:
    dem = names
for r, d in zip(rows, dem):
    d = re.sub(r"qdpb::", "", d)
    d = re.sub(r"\(.*\)$", "", d)
    print(f"{r.get('regs', '?'):>4} regs  stack {r.get('stack', 0):>5}  spill {r.get('spill_st', 0):>4}/{r.get('spill_ld', 0):<4} {d}")
