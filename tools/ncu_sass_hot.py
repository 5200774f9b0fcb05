"""Hottest SASS instructions of one kernel (first launch in the report), with stall-sample share.

    python tools/ncu_sass_hot.py report.ncu-rep kernel_name [n] [context]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
c = h.index("Warp Stall Sampling (All Samples)")
d = []
for r in rows[hi + 1:]:
    try:
        d.append((float(r[c] or 0), r[1].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in d) or 1
print(f"{len(d)} instructions")
top = sorted(range(len(d)), key=lambda i: -d[i][0])[:n]
for i in sorted(top):
    lo = max(0, i - ctx)
    for j in range(lo, i + 1):
        mark = "*" if j == i else " "
        print(f"{mark}{j:6d} {100 * d[j][0] / tot:5.1f}%  {d[j][1]}")
