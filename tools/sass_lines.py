"""Dev tool: dynamic instruction counts per source line for one kernel.
Joins an ncu source-page SASS csv (Instructions Executed per address) with nvdisasm -g
line info.  Usage: python tools/sass_lines.py NCU_SASS_CSV NVDISASM_OUT KERNEL_SUBSTR MANGLED_PREFIX UNITS [COLUMN]
(COLUMN defaults to "Instructions Executed"; e.g. "Warp Stall Sampling (All Samples)", "stall_long_sb")."""
import collections
import csv
import re
import sys


def main(csv_path, sass_path, kname, mangled, units, col="Instructions Executed", top=40):
    rows = list(csv.reader(open(csv_path)))
    secs, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            secs.append(cur)
            continue
        if cur is not None:
            cur["rows"].append(r)
    sec = [s for s in secs if kname in s["name"]][0]
    h, data = sec["rows"][0], sec["rows"][1:]
    ia, iex = h.index("Address"), h.index(col)
    base = min(int(r[ia], 16) for r in data)
    ex = {int(r[ia], 16) - base: float(r[iex] or 0) for r in data}
    lines, curl, inside = {}, None, False
    for line in open(sass_path):
        if line.startswith(".text." + mangled):
            inside = True
            continue
        if inside and line.startswith("//--------------------- .text."):
            break
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            curl = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m and curl:
            lines[int(m.group(1), 16)] = curl
    cnt = collections.Counter()
    for off, e in ex.items():
        cnt[lines.get(off, ("?", 0))] += e
    tot = sum(cnt.values())
    print(f"total {tot:.0f} = {tot / units:.1f} per unit")
    for (f, l), c in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
        src = ""
        try:
            src = open("paper_1709_08990_b200/csrc/" + f).read().split("\n")[l - 1].strip()[:90]
        except Exception:
            pass
        print(f"{c / units:7.1f} {f}:{l}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], float(sys.argv[5]), *sys.argv[6:7])
