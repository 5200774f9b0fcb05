set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cat MEASURED_PEAKS.json
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc=$?
timeout 600 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench rc=$?
timeout 600 python bench.py --sweep config5_qwen --no-cpu-baseline > gpurun_out/bench_c5q.json 2> gpurun_out/bench_c5q.err; echo benchq rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_v14.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_cells -s 1 -c 1 -o gpurun_out/prof_v14 python tools/profile_run.py gpt-oss-120b 100 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
cat gpurun_out/bench_c5.json gpurun_out/bench_c5q.json
