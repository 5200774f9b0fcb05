"""Hottest CUDA source lines of one kernel in an ncu report (warp-stall samples per line).

    python tools/ncu_hot.py report.ncu-rep kernel_name [n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
per_line = defaultdict(float)
text = {}
fname = ""
col = None
tot = 0.0
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        col = r.index("Warp Stall Sampling (All Samples)")
        continue
    if col is None or len(r) <= col:
        continue
    try:
        s = float(r[col] or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    per_line[key] += s
    text.setdefault(key, r[1][:120])
    tot += s
for (f, line), s in sorted(per_line.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * s / max(tot, 1):5.1f}%  {f}:{line:<5} {text[(f, line)]}")
