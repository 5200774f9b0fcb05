"""Per-kernel evidence table from one `ncu --set full` report (first launch of each kernel).

    python tools/ncu_table.py gpurun_out/prof_all_v19.ncu-rep [peak_gbs] > profiles/r1_ncu_kernels_v19.md

Columns: duration, DRAM GB/s and % of the HBM peak, L2 GB/s, SM throughput,
FP64 pipe activity, achieved occupancy, warp efficiency (active threads per
executed instruction, of 32) and the dominant stall reason.
"""

import csv
import io
import subprocess
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--json=")]
json_out = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--json=")), None)
rep = args[0]
peak = float(args[1]) if len(args) > 1 else 6553.6
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {n: i for i, n in enumerate(hdr)}


def val(r, name, scale=1.0):
    i = col.get(name)
    if i is None or not r[i].strip():
        return None
    try:
        return float(r[i].replace(",", "")) * scale
    except ValueError:
        return None


def unit_scale(name, to):
    u = units[col[name]] if name in col else ""
    table = {"byte/second": 1e-9, "Kbyte/second": 1e-6, "Mbyte/second": 1e-3, "Gbyte/second": 1.0,
             "Tbyte/second": 1e3, "B/s": 1e-9, "KB/s": 1e-6, "MB/s": 1e-3, "GB/s": 1.0, "Tbyte/s": 1e3,
             "Gbyte/s": 1.0, "Mbyte/s": 1e-3, "Kbyte/s": 1e-6, "byte/s": 1e-9, "TB/s": 1e3,
             "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
             "sector/ns": 32.0, "sector/us": 32e-3, "sector/ms": 32e-6, "sector/s": 32e-9}
    return table.get(u, 1.0)


stall_cols = [n for n in hdr if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith(".ratio")]
seen = set()
table = {}
print(f"# Per-kernel ncu evidence ({rep.split('/')[-1]}; first launch of each kernel; HBM peak {peak:.0f} GB/s)\n")
print("| kernel | µs | DRAM GB/s | % HBM peak | L2 GB/s | SM % | FP64 pipe % | occupancy % | warp eff. (of 32) | top stall (cycles per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in data:
    name = r[col["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    if name in seen:
        continue
    seen.add(name)
    dur = val(r, "gpu__time_duration.sum", unit_scale("gpu__time_duration.sum", "us"))
    dram = val(r, "dram__bytes.sum.per_second", unit_scale("dram__bytes.sum.per_second", "GB/s"))
    l2 = val(r, "lts__t_sectors.sum.per_second", unit_scale("lts__t_sectors.sum.per_second", "GB/s"))
    sm = val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
    fp64 = val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
    occ = val(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
    eff = val(r, "smsp__thread_inst_executed_per_inst_executed.ratio")
    best, bname = -1.0, ""
    for n in stall_cols:
        v = val(r, n)
        if v is not None and v > best and "selected" not in n:
            best, bname = v, n.split("stalled_")[-1].replace("_per_issue_active.ratio", "") + f" ({v:.1f})"
    issue = val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active")
    table[name] = {"us": dur, "dram_gbs": dram, "dram_frac_of_peak": None if dram is None else dram / peak,
                   "l2_gbs": l2, "sm_pct": sm, "fp64_pipe_pct": fp64, "warps_active_pct": occ,
                   "issue_active_pct": issue, "active_threads_per_warp": eff, "top_stall": bname,
                   "dram_bytes": sum((val(r, n) or 0) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(
                       units[col[n]] if n in col else "byte", 1) for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))}
    f = lambda x, d=1: "–" if x is None else f"{x:.{d}f}"
    print(f"| {name} | {f(dur)} | {f(dram, 0)} | {f(None if dram is None else 100 * dram / peak)} | {f(l2, 0)} | "
          f"{f(sm)} | {f(fp64)} | {f(occ)} | {f(eff)} | {bname} |")

if json_out:
    import json

    with open(json_out, "w") as fh:
        json.dump({"source": rep.split("/")[-1], "hbm_peak_gbs": peak, "kernels": table}, fh, indent=1)
