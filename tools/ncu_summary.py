"""Summarise ncu captures into profiles/ (markdown + json).

    python tools/ncu_summary.py gpurun_out/prof_v4.ncu-rep gpurun_out/launches_v4.csv profiles/r1_ncu_v4

Reads the `--set full` report for per-kernel speed-of-light, occupancy, stall
and DRAM figures, and the `--metrics gpu__time_duration.sum[,dram__bytes_*]`
launch list for each kernel's share of a bench step (cold-cache, serialised
launches: compare shares, not absolute times).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

WANT = [
    ("Duration", "ms"), ("Compute (SM) Throughput", "%"), ("Memory Throughput", "%"), ("DRAM Throughput", "%"),
    ("Issue Slots Busy", "%"), ("Achieved Occupancy", "%"), ("Registers Per Thread", ""),
    ("Warp Cycles Per Issued Instruction", "cycle"), ("Avg. Active Threads Per Warp", ""),
    ("L2 Hit Rate", "%"), ("L1/TEX Hit Rate", "%"),
]
RAW = [
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_local_ld.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu_csv(args: list[str]) -> list[list[str]]:
    out = subprocess.run(["ncu", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def kernels_in(rep: str) -> list[str]:
    rows = ncu_csv(["-i", rep, "--page", "details"])
    h = rows[0]
    k = h.index("Kernel Name")
    seen = []
    for r in rows[1:]:
        name = r[k].split("(")[0].replace("<unnamed>::", "")
        if name not in seen:
            seen.append(name)
    return seen


def details(rep: str, kernel: str) -> dict:
    rows = ncu_csv(["-i", rep, "--page", "details", "-k", f"regex:{kernel}$|{kernel}\\("])
    if not rows:
        return {}
    h = rows[0]
    idx = {n: i for i, n in enumerate(h)}
    out = {}
    for r in rows[1:]:
        n = r[idx["Metric Name"]]
        if n in dict(WANT) and n not in out:
            out[n] = r[idx["Metric Value"]] + (" " + r[idx["Metric Unit"]] if r[idx["Metric Unit"]] else "")
    raw = ncu_csv(["-i", rep, "--page", "raw", "-k", f"regex:{kernel}$|{kernel}\\("])
    if len(raw) >= 3:
        h, units, v = raw[0], raw[1], raw[2]
        for n in RAW:
            if n in h:
                i = h.index(n)
                out[n] = (v[i] + " " + units[i]).strip()
        stalls = []
        for i, n in enumerate(h):
            if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out["top_stalls_cycles_per_issue"] = {n: round(x, 2) for x, n in stalls[:5]}
    return out


def launch_shares(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    idx = {n: i for i, n in enumerate(h)}
    agg = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    seen_ids = defaultdict(set)
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        name = r[idx["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
        metric, val = r[idx["Metric Name"]], float(r[idx["Metric Value"]] or 0)
        if r[idx["ID"]] not in seen_ids[name]:
            seen_ids[name].add(r[idx["ID"]])
            agg[name]["launches"] += 1
        if metric == "gpu__time_duration.sum":
            agg[name]["ms"] += val / 1e6
        elif metric.startswith("dram__bytes"):
            agg[name]["dram_bytes"] += val
    total = sum(v["ms"] for v in agg.values())
    for v in agg.values():
        v["share"] = v["ms"] / total if total else 0.0
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))


def main() -> int:
    rep, launches, out = sys.argv[1], sys.argv[2], Path(sys.argv[3])
    data = {"report": rep, "launch_list": launches, "kernels": {}, "shares": launch_shares(launches)}
    for k in kernels_in(rep):
        data["kernels"][k] = details(rep, k)
    out.with_suffix(".json").write_text(json.dumps(data, indent=2) + "\n")
    lines = [f"# ncu summary ({Path(rep).name}, {Path(launches).name})", "",
             "## Share of one bench step (launch list; cold, serialised)", "",
             "| kernel | launches | ms | share | DRAM bytes |", "|---|---|---|---|---|"]
    for k, v in data["shares"].items():
        lines.append(f"| {k} | {v['launches']} | {v['ms']:.3f} | {100 * v['share']:.1f}% | {v['dram_bytes']:.3e} |")
    lines += ["", "## Per-kernel (`--set full`, first captured launch)", ""]
    for k, d in data["kernels"].items():
        lines.append(f"### {k}")
        for n, _ in WANT:
            if n in d:
                lines.append(f"- {n}: {d[n]}")
        for n in RAW:
            if n in d:
                lines.append(f"- `{n}`: {d[n]}")
        if "top_stalls_cycles_per_issue" in d:
            lines.append(f"- top stalls (cycles/issue): {d['top_stalls_cycles_per_issue']}")
        lines.append("")
    out.with_suffix(".md").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    return 0


if __name__ == "__main__":
    sys.exit(main())
