"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki][:60] + ((" " + r[gi]) if gi is not None else "")
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total {tot / 1e3:.1f} us over {sum(n for n, _ in agg.values())} launches")
for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v / 1e3:10.1f} us {100 * v / tot:5.1f}%  n={n:5d}  avg={v / n / 1e3:8.2f} us  {k}")
