"""Top SASS lines of an exported `ncu --page source --csv --print-source sass` by stall samples.

    python tools/sass_hot.py gpurun_out/prof_x_sass.csv [N] [stall_column]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
h = rows[hi]
ix = {k: i for i, k in enumerate(h)}
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
tot = collections.Counter()
for r in body:
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            tot[k] += int(r[ix[k]] or 0)
print("totals:", dict(tot.most_common(10)))
ops = collections.Counter()
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
print("warp-instr by opcode:", ops.most_common(14))
body.sort(key=lambda r: -int(r[ix[col]] or 0))
for r in body[:n]:
    top = sorted(((int(r[ix[k]] or 0), k) for k in h if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:2]
    print(r[ix[col]], r[ix["Instructions Executed"]], r[ix["Source"]].strip()[:70], top)
