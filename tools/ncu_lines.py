"""Executed instructions and stall samples of one kernel per CUDA source line:
the ncu SASS page (per-instruction counters) joined by offset with the line
table nvdisasm prints for the same binary.

    python tools/ncu_lines.py report.ncu-rep kernel_substring [n] [--so path]

Needs the .so the report was captured with (default: the in-tree build).
"""

from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from sass_spills import SO, disassemble  # noqa: E402


def line_table(lines: list[str]) -> dict[int, str]:
    src, out = "?", {}
    for line in lines:
        if "//##" in line:
            m = re.search(r"line (\d+)", line)
            f = re.search(r'"([^"]+)"', line)
            if m:
                src = (f.group(1).split("/")[-1] if f else "?") + ":" + m.group(1)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", line)
        if m:
            out[int(m.group(1), 16)] = src
    return out


def main() -> None:
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    so = Path(sys.argv[sys.argv.index("--so") + 1]) if "--so" in sys.argv else SO
    if "--so" in sys.argv:
        args.remove(str(so))
    rep, kern = args[0], args[1]
    n = int(args[2]) if len(args) > 2 else 30
    funcs = disassemble(so)
    name = next(k for k in funcs if kern in k)
    table = line_table(funcs[name])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    inst, samp = collections.Counter(), collections.Counter()
    for r in data:
        off = int(r[ia], 16) - base
        src = table.get(off, "?")
        inst[src] += float(r[ie] or 0)
        samp[src] += float(r[isamp] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"{name[:80]}: {ti:.4g} warp instructions, {ts:.4g} stall samples")
    print(f"{'line':28s} {'inst %':>7s} {'stall %':>8s}")
    for src, v in inst.most_common(n):
        print(f"{src:28s} {100 * v / ti:7.2f} {100 * samp[src] / ts:8.2f}")


if __name__ == "__main__":
    main()
