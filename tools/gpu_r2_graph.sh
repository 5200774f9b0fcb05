mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/configs_timing.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo cfg_rc=$?
python -c "
import json; d=json.load(open('gpurun_out/configs.json'))
for c in d['configs']: print(c['config'], c['candidates'], 'direct', round(c['device_pipeline_direct_ms'],3), 'graph', round(c['device_pipeline_graph_ms'],3), 'search', round(c['device_search_ms'],3), 'json', round(c['run_search_json_ms'],3))"
for g in 0 1; do
  if [ $g = 1 ]; then export LC_NO_GRAPH=1; fi
  timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_g$g.json 2> gpurun_out/bench_g$g.err; echo bench_rc=$?
  python -c "
import json; d=json.loads(open('gpurun_out/bench_g$g.json').read().strip().splitlines()[-1])
print('graph_off=$g', 'ms', round(d['ms_per_step'],3), 'e2e_ms', round(d['search_wall_ms']['e2e'],3), 'ns ms', round(d['north_star']['ms_per_step'],3), 'ns e2e', round(d['north_star']['e2e_ms_per_step'],3))"
done
