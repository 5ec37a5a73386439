"""Registers / spills per kernel from build/akv/build.log (ptxas -v), demangled.

    python tools/regs.py [filter]
"""
import re
import subprocess
import sys

log = open("build/akv/build.log").read().splitlines()
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur, spill = None, ""
rows = []
for line in log:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
        cur = None
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for (mg, r, sp), nm in zip(rows, names):
    nm = re.sub(r"\(.*", "", nm).replace("void ", "")
    if flt in nm:
        print(f"{r:4d} {sp:16s} {nm}")
