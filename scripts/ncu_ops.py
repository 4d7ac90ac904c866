"""Executed-instruction mix (by opcode) and the hottest SASS lines of an ncu report."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
k = h.index("Instructions Executed")
agg, tot, lines = collections.Counter(), 0.0, []
for r in rows[2:]:
    if len(r) <= k or not r[0].startswith("0x"):
        continue
    try:
        v = float(r[k])
    except ValueError:
        continue
    toks = r[1].strip().split()
    op = toks[1] if toks[0].startswith("@") else toks[0]
    agg[op.split(".")[0]] += v
    tot += v
    lines.append((v, r[1].strip()))
print(f"total warp instructions {tot:.0f}")
for op, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"  {op:12s} {100 * v / tot:5.1f}%")
