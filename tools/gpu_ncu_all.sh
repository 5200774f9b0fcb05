mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_qtables|k_dstables|k_dseries|k_expand|k_tails|k_front_pass1|k_pools_partial|k_front_final|k_disagg|k_enum_flags|k_scatter" -s 11 -c 11 -o gpurun_out/prof_all_v15 python tools/profile_run.py deepseek-v3 100 > gpurun_out/ncu_all.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu_all.log
