# full GPU check: every -m gpu test, smoke, the bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("ms", d["ms_per_step"], "e2e_ms", d["search_wall_ms"]["e2e"], "frac", d["roofline"]["frac"])
print("kernel_ms", {k: round(v, 3) for k, v in d["roofline"]["kernel_ms"].items()})
ns = d.get("north_star") or {}
print("north_star ms", ns.get("ms_per_step"), "e2e", ns.get("e2e_ms_per_step"))
PY
tail -3 gpurun_out/bench.err
