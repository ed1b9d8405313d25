"""Dev tool: per-source-file totals of a column of an ncu SASS source page (see sass_lines.py).
Usage: python tools/sass_files.py NCU_SASS_CSV NVDISASM_OUT KERNEL_SUBSTR MANGLED UNITS [COLUMN]"""
import collections
import contextlib
import io
import sys

sys.path.insert(0, "tools")
import sass_lines  # noqa: E402

buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    sass_lines.main(*sys.argv[1:5], float(sys.argv[5]), *sys.argv[6:7], top=100000)
agg = collections.Counter()
for line in buf.getvalue().splitlines()[1:]:
    parts = line.split()
    agg[parts[1].split(":")[0]] += float(parts[0])
for k, v in agg.most_common():
    print(f"{v:9.1f} {k}")
