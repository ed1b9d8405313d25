"""Dev tool: headline counters and stall reasons of each kernel in an ncu report.
Usage: python tools/ncu_stalls.py REPORT.ncu-rep [KERNEL_SUBSTR]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]
for r in rows[2:]:
    d = dict(zip(h, r))
    if sub not in d["Kernel Name"]:
        continue
    print(d["Kernel Name"][:90])
    for k in KEYS:
        print(f"   {k:60s} {d.get(k)}")
    st = [(k, float(d[k] or 0)) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    for k, v in sorted(st, key=lambda kv: -kv[1])[:9]:
        print(f"   stall {k[len('smsp__pcsamp_warps_issue_stalled_'):]:28s} {v / tot:.3f}")
