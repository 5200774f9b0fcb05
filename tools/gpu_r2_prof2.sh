mkdir -p gpurun_out
bash tools/gpu_kernel_variants.sh
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_eval_cells|k_dseries|k_tails|k_qtables|k_front_final|k_pools_partial" -c 6 -o gpurun_out/prof_r2h2 python tools/profile_run.py gpt-oss-120b 100 > gpurun_out/ncu_r2h2.log 2>&1; echo ncu_rc=$?
tail -2 gpurun_out/ncu_r2h2.log
