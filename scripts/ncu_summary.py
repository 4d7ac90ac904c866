"""Key metrics + top stall reasons + hottest SASS lines of an ncu --set full report."""
import csv
import io
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1], *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
h, units, rows = raw[0], raw[1], raw[2:]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum"]
for ri, r in enumerate(rows):
    print(f"--- kernel {ri}: {r[h.index('Kernel Name')][:90]}")
    for k in keys:
        if k in h:
            print(f"   {k:70s} {r[h.index(k)]} {units[h.index(k)]}")
    st = []
    for i, name in enumerate(h):
        if "pcsamp_warps_issue_stalled" in name and not name.endswith("not_issued"):
            try:
                st.append((float(r[i]), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source", "sass"]))))
tab = [r for r in src if len(r) > 5 and r[0].startswith("0x")]
tot = sum(int(r[2] or 0) for r in tab) or 1
print("   hottest SASS:")
for r in sorted(tab, key=lambda r: -int(r[2] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    print(f"     {100 * int(r[2]) / tot:5.1f}%  {r[1].strip()[:100]}")
