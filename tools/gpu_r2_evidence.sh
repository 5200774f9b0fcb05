# Long parity campaign and the bench's own ncu launch list at HEAD
mkdir -p gpurun_out
LC_FUZZ_N=3000 LC_FUZZ_BATCHES=300 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_fuzz_long.log 2>&1; echo fuzz_rc=$?
tail -3 gpurun_out/pytest_fuzz_long.log
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 150 \
  --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --north-star none \
  > gpurun_out/bench_under_ncu.log 2>&1; echo ncu_launch_rc=$?
