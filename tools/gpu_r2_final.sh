# Round-2 evidence at HEAD: GPU tests + smoke, the default bench line, per-model launch lists with
# DRAM bytes (K2 traffic), one ncu --set full of the main kernels, the north-star sweep bench.
#   bash tools/gpu_r2_final.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu_${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo bench_rc=$?
for m in gpt-oss-120b deepseek-v3; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/lt_${m}.csv python tools/profile_run.py $m 100 > /dev/null 2>&1; echo lt_${m}_rc=$?
done
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_eval_cells|k_pools_partial|k_front_pass3|k_front_final|k_qtables|k_dstables|k_dseries|k_ptables|k_tails|k_disagg|k_scatter_fit|k_front_mid" \
  -c 24 -o gpurun_out/prof_${tag} python tools/profile_run.py gpt-oss-120b 100 > gpurun_out/ncu_${tag}.log 2>&1; echo ncu_full_rc=$?
LC_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
  --csv --log-file gpurun_out/launches_bench_${tag}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --north-star none \
  > gpurun_out/bench_under_ncu_${tag}.log 2>&1; echo ncu_launch_rc=$?
