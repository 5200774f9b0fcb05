# the bench's own ncu launch list (direct launches: LC_NO_GRAPH=1, the same kernels the graph holds),
# plus the diagnostics of tools/gpu_diag.sh
mkdir -p gpurun_out
LC_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
  --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --north-star none \
  > gpurun_out/bench_under_ncu.log 2>&1; echo ncu_launch_rc=$?
tail -3 gpurun_out/bench_under_ncu.log
bash tools/gpu_diag.sh
