"""Dev tool: key metrics of every kernel in an ncu report.  Usage: python tools/ncu_summary.py REP"""
import csv
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
for row in rows[2:]:
    print(row[h.index("Kernel Name")][:70])
    for k in KEYS:
        if k in h:
            print(f"   {k:60s} {row[h.index(k)]} {units[h.index(k)]}")
    st = [(k, row[i]) for i, k in enumerate(h) if "average_warps_issue_stalled" in k and "per_issue_active" in k]
    st = sorted(((float(v or 0), k.split("stalled_")[1].split("_per")[0]) for k, v in st), reverse=True)[:6]
    print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st))
