"""Dev tool: profiles/traffic.json from cold ncu launch lists of bench.py runs, one per
workload (launches_<tag>_<cfg>.csv): DRAM bytes (read + write) per call of each phase,
summed over the phase's kernels (kernels assigned to a phase by name).
Usage: python tools/traffic_json.py TAG DIR"""
import collections
import csv
import json
import sys
from pathlib import Path

ENC = ("encode", "size_scan", "sizes")
tag, d = sys.argv[1], Path(sys.argv[2])
out = {"_note": f"DRAM bytes (read + write) per call of each phase, summed over its kernels, from the cold-cache "
                f"ncu launch lists profiles/r02/launches_{tag}_<cfg>.csv (bench.py --workload <cfg> --steps 2 "
                f"--warmup 3, per-kernel averages over the launches); ncu flushes caches before every kernel, so "
                f"writes still dirty in L2 at kernel end are not counted"}
for cfg in ("cfg2", "cfg3", "cfg4", "cfg5"):
    p = d / f"launches_{tag}_{cfg}.csv"
    if not p.exists():
        continue
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for (_, k), m in per.items():
        if not k.startswith("void bcgpu::") and not k.startswith("bcgpu::"):
            continue
        agg[k][0] += 1
        agg[k][1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    for phase in ("encode", "decode"):
        tot = 0.0
        for k, (c, b) in agg.items():
            name = k.split("(")[0]
            is_enc = any(e in name for e in ENC)
            if (phase == "encode") == is_enc:
                tot += b / c
        out[f"{cfg}:{phase}"] = int(tot)
print(json.dumps(out, indent=1))
