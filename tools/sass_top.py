"""Instruction mix, stall totals and the hottest SASS lines per kernel of an
`ncu --page source --csv --print-source sass` export.

    python tools/sass_top.py gpurun_out/prof_x_sass.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
starts = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r]
for si, st in enumerate(starts):
    h = rows[st]
    ix = {k: i for i, k in enumerate(h)}
    end = starts[si + 1] if si + 1 < len(starts) else len(rows)
    body = [r for r in rows[st + 1:end] if len(r) == len(h)]
    ops, stall, tot = collections.Counter(), collections.Counter(), 0
    for r in body:
        s = r[ix["Source"]].split()
        if not s:
            continue
        op = s[1] if s[0].startswith("@") else s[0]
        n = int(r[ix["Instructions Executed"]] or 0)
        ops[op.split(".")[0]] += n
        tot += n
        for k in h:
            if k.startswith("stall_") and "Not Issued" not in k:
                stall[k] += int(r[ix[k]] or 0)
    print(rows[st - 1][:2] if st else "", "warp-instr", tot)
    print("  ops:", ops.most_common(16))
    print("  stalls:", stall.most_common(10))
    col = "Warp Stall Sampling (All Samples)"
    body.sort(key=lambda r: -int(r[ix[col]] or 0))
    for r in body[:N]:
        print("   ", r[ix[col]], r[ix["Address"]], r[ix["Source"]][:100])
