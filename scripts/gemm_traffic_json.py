"""profiles/<tag>/ncu_gemm_traffic.json from scripts/ncu_round.sh's step GEMM
capture (ncu --csv metrics of one decode step's 37 tc_gemm launches): DRAM
bytes (read + write) and duration per launch. Usage: gemm_traffic_json.py
<step_gemms.csv> <out.json> <what>"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
hdr = rows[hdr_i]
iid, ik, im, iv = (hdr.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
per = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= iv:
        continue
    e = per.setdefault(int(r[iid]), {"kernel": r[ik][:60]})
    e[r[im]] = float(r[iv].replace(",", "")) if r[iv].replace(",", "").replace(".", "").isdigit() else r[iv]
out = []
for i, e in sorted(per.items()):
    out.append({"id": i, "kernel": e["kernel"],
                "dram_bytes": e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0),
                "us": e.get("gpu__time_duration.sum"), "grid": str(e.get("launch__grid_size"))})
mean = sum(o["dram_bytes"] for o in out) / max(len(out), 1)
json.dump({"what": sys.argv[3], "launches": len(out), "bytes_per_launch_mean": mean,
           "per_launch": out}, open(sys.argv[2], "w"), indent=1)
print(len(out), mean)
