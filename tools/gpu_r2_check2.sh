# GPU tests, e2e host phases and the bench line (round-2 host-path changes)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
LC_HOST_TIMING=1 timeout 300 python tools/e2e_timing.py > gpurun_out/e2e_timing4.txt 2>&1; tail -7 gpurun_out/e2e_timing4.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_check2.json 2> gpurun_out/bench_check2.err; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_check2.json").read().strip().splitlines()[-1])
ns = d["north_star"]
print("ms", round(d["ms_per_step"], 3), "e2e", round(d["search_wall_ms"]["e2e"], 3), "ns", round(ns["ms_per_step"], 3), round(ns["e2e_ms_per_step"], 3))
PY
