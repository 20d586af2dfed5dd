"""Registers / spills per kernel instance from `nvcc -Xptxas -v` output
(stdin):  nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_summary.py"""
import re
import subprocess
import sys

cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and "spill" not in cur:
        cur["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = [r["name"] for r in rows]
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for r, d in zip(rows, dem):
    d = re.sub(r"lfb::\(anonymous namespace\)::", "", d)
    d = d.split("(")[0]
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', '?'):>9}  {d}")
