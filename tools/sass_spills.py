"""Per-kernel SASS census of the built engine: instruction count, local-memory
spills (STL/LDL) attributed to source lines, generic vs shared loads, calls.

    python tools/sass_spills.py [kernel-substring ...]

Reads paper_2601_06288_b200/_lc_b200.so (built with -lineinfo), no GPU needed.
"""

from __future__ import annotations

import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SO = ROOT / "paper_2601_06288_b200" / "_lc_b200.so"


def disassemble(so: Path = SO) -> dict[str, list[str]]:
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", str(Path(so).resolve())], cwd=td, check=True, capture_output=True)
        cubin = next(Path(td).glob("*.cubin"))
        txt = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], check=True, capture_output=True,
                             text=True).stdout
    funcs: dict[str, list[str]] = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"^\.text\.(\S+):", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur is not None:
            funcs[cur].append(line)
    return funcs


def census(lines: list[str]) -> dict:
    src = None
    stl, ldl = collections.Counter(), collections.Counter()
    ops = collections.Counter()
    for line in lines:
        if "//##" in line:
            m = re.search(r'line (\d+)', line)
            f = re.search(r'"([^"]+)"', line)
            if m:
                src = (f.group(1).split("/")[-1] if f else "?") + ":" + m.group(1)
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        base = op.split(".")[0]
        ops[base] += 1
        if base == "STL":
            stl[src] += 1
        elif base == "LDL":
            ldl[src] += 1
    return {"n": sum(ops.values()), "ops": ops, "stl": stl, "ldl": ldl}


def main(argv: list[str]) -> None:
    funcs = disassemble()
    pats = argv or [""]
    for name, lines in funcs.items():
        short = re.sub(r"_ZN\d+_GLOBAL__N__\w+?_cu_\w{8}\d+", "", name)
        if not any(p in name for p in pats):
            continue
        c = census(lines)
        o = c["ops"]
        print(f"{short[:70]}: {c['n']} instr, STL {o['STL']} LDL {o['LDL']} LD {o['LD']} LDS {o['LDS']} "
              f"LDG {o['LDG']} CALL {o['CALL']} DADD {o['DADD']} DMUL {o['DMUL']} DFMA {o['DFMA']}")
        if argv:
            print("   STL by line:", c["stl"].most_common(12))
            print("   LDL by line:", c["ldl"].most_common(12))


if __name__ == "__main__":
    main(sys.argv[1:])
