# round-2 GPU check: sweep-scale parity + NCCL skip + bench (headline + north star)
set -x
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_nccl.py -x -q > gpurun_out/pytest_sweep.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_sweep.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
