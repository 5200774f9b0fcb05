# GPU tests, the default bench line, configs 1-4 timing and the strong-scaling projection
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_misc.json 2> gpurun_out/bench_misc.err; echo bench_rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_misc.json").read().strip().splitlines()[-1])
ns = d["north_star"]
print("ms", round(d["ms_per_step"], 3), "e2e", round(d["search_wall_ms"]["e2e"], 3), "ns", round(ns["ms_per_step"], 3), round(ns["e2e_ms_per_step"], 3), "frac", round(d["roofline"]["frac"], 3), "traffic", d["roofline"].get("traffic"))
PY
timeout 600 python tools/configs_timing.py > gpurun_out/configs1to4.json 2> gpurun_out/configs.err; echo configs_rc=$?
timeout 600 python tools/shard_projection.py > gpurun_out/shard_projection.txt 2>&1; echo shard_rc=$?; cat gpurun_out/shard_projection.txt | tail -5
