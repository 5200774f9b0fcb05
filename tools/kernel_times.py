"""Per-kernel µs from an ncu launch list (gpu__time_duration.sum): mean over launches per kernel name.

    python tools/kernel_times.py gpurun_out/launches_x.csv [...]
"""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    t = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        t[name].append(v / 1000.0 if unit in ("nsecond", "ns") else v)
    tot = sum(sum(v) / len(v) for v in t.values())
    print(f"== {path}: sum of per-kernel means {tot:.1f} us")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        print(f"  {k:28s} {sum(v) / len(v):9.1f} us  x{len(v)}")
