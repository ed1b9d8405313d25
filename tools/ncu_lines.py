"""Dev tool: top source lines (by executed warp instructions) and opcode mix of one kernel
in an ncu report.  Usage: python tools/ncu_lines.py REPORT.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__grid_size", "launch__occupancy_limit_shared_mem"]
for row in r[2:]:
    print(row[h.index("Kernel Name")][:90] if "Kernel Name" in h else "")
    for k in keys:
        if k in h:
            print(f"   {k:70s} {row[h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
cur = None
hdr = None
res = []
ops = collections.Counter()
for x in rows:
    if len(x) == 2 and x[0] == "File Path":
        cur = x[1].split("/")[-1]
        continue
    if x and x[0] == "Line No":
        hdr = x
        continue
    if not hdr or len(x) < 9:
        continue
    try:
        e = int(x[7] or 0)
        s = int(x[4] or 0)
    except ValueError:
        continue
    if x[0]:
        res.append((e, s, cur, x[0], x[1][:100]))
    else:
        op = x[3].split()
        if op:
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            ops[o.split(".")[0]] += e
tot = sum(v[0] for v in res) or 1
print("executed warp instructions:", tot)
for e, s, f, ln, t in sorted(res, reverse=True)[:top]:
    print(f"{e / tot:6.3f} {s:7d} {f}:{ln} {t}")
t2 = sum(ops.values()) or 1
print("opcode mix:", ", ".join(f"{o} {c / t2:.3f}" for o, c in ops.most_common(16)))
