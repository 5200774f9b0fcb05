# ncu evidence for round 2: one --set full capture of the main kernels (GPT-OSS-120B batch of
# 100 config-5 searches) and the launch list of a short bench run.
#   bash tools/gpu_r2_profile.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:k_eval_cells|k_pools_partial|k_front_pass|k_front_final|k_qtables|k_dstables|k_dseries|k_ptables|k_tails|k_disagg|k_scatter_fit|k_front_mid" \
  -c 24 -o gpurun_out/prof_${tag} python tools/profile_run.py gpt-oss-120b 100 > gpurun_out/ncu_${tag}.log 2>&1; echo ncu_full_rc=$?
tail -3 gpurun_out/ncu_${tag}.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --north-star none > gpurun_out/bench_under_ncu_${tag}.log 2>&1; echo ncu_launch_rc=$?
