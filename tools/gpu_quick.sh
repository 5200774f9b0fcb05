# quick correctness + timing check: sweep/parity/sharded GPU tests and a config5 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_quick.txt 2>&1; echo tests rc=$?
tail -3 gpurun_out/pytest_quick.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_quick.json'))
print('ms/step', round(d['ms_per_step'],3), 'e2e ms', round(d['search_wall_ms']['e2e'],3), 'seq', round(d['search_wall_ms']['per_model_sequential_device'],3))
print({k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})"
