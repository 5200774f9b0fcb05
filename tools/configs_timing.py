"""Search wall time for BASELINE configs 1-4, one B200.

For each config: the device search to fronts + best + counts on the host
(Engine.run_batch + fetch_fronts), the full report JSON (run_search_json) and
the object report (run_search + to_json), medians over repeated runs; beside
them the CPU oracle (C restatement, one thread) on this box and the pure-Python
reference's wall time recorded when the golden report was made
(tests/golden/reports/*: _meta.reference_wall_s, survey container CPU).

    python tools/configs_timing.py > profiles/r2_configs1to4.json
"""

import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

import paper_2601_06288_b200 as pkg  # noqa: E402
from golden_io import BY_NAME, db_path, golden_report, hw_docs, model_doc  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2601_06288_b200.engine import fetch_fronts, get_engine  # noqa: E402
from product_cases import case_objects  # noqa: E402

NAMES = ["cfg1_qwen3_agg", "cfg2_qwen3_disagg", "cfg3_llama70b_kv50", "cfg3_llama70b_kv70", "cfg3_llama70b_kv90",
         "cfg4_dsv3"]
REPS = 20


def med(fn, reps=REPS):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1000.0)
    return statistics.median(ts)


out = []
eng = get_engine(0)
for name in NAMES:
    case = BY_NAME[name]
    db, model, workload, space, dc = case_objects(case)

    def summary():
        with eng._lock:
            o = eng.run_batch(db, model, space, [workload], dc)
            fetch_fronts(o)
        return o

    for _ in range(3):
        o = summary()
        pkg.run_search_json(db, model, workload, space, disagg_constants=dc)
    t_sum = med(summary)
    t_json = med(lambda: pkg.run_search_json(db, model, workload, space, disagg_constants=dc))
    t_obj = med(lambda: pkg.run_search(db, model, workload, space, disagg_constants=dc).to_json())
    header, recs = oracle.read_db_records(db_path(case))
    header, recs = oracle.mutate(header, recs, case.get("mutation"), hw_docs())
    t_orc = med(lambda: oracle.run_search(header, recs, model_doc(case["model"]), case["workload"], case.get("space"),
                                          case.get("disagg"), case.get("extrapolation", "default")), reps=3)
    g = golden_report(name)
    # device time of the K0..K4 pipeline alone: direct launches (lc_replay_last, CUDA events per stage)
    # and the batch's CUDA graph relaunched (lc_replay_async between events on the engine stream)
    import torch

    with eng._lock:
        o = eng.run_batch(db, model, space, [workload], dc)
        t_direct = statistics.median(float(sum(eng.replay(1).kernel_ms)) for _ in range(REPS))
        st = torch.cuda.ExternalStream(eng.stream_ptr())
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            eng.replay_async()
        a.record(st)
        for _ in range(REPS):
            eng.replay_async()
        b.record(st)
        b.synchronize()
        t_graph = a.elapsed_time(b) / REPS
    out.append({"config": name, "candidates": int(o.results[0]["n_enumerated"]), "rows": g["counts"]["evaluated"],
                "device_pipeline_direct_ms": t_direct, "device_pipeline_graph_ms": t_graph,
                "device_search_ms": t_sum, "run_search_json_ms": t_json, "run_search_objects_to_json_ms": t_obj,
                "cpu_oracle_1thread_ms": t_orc, "python_reference_ms": 1000.0 * g["_meta"]["reference_wall_s"]})
print(json.dumps({"reps": REPS, "note": "median wall ms; python_reference_ms from the golden generator (CPU, survey "
                                        "container); device_search_ms = run_batch + fetch_fronts (fronts, best, counts)",
                  "configs": out}, indent=1))
