"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        per[(int(r[ii]), r[ki][:70])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (_, k), m in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} n={a[0]:3d} avg_us={a[1] / a[0] / 1000:8.2f} rdMB={a[2] / a[0] / 1e6:8.1f} wrMB={a[3] / a[0] / 1e6:8.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
