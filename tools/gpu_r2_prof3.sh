# per-kernel A/B of variants/*.so, stream settings, the e2e breakdown and one ncu --set full of k_eval_cells
mkdir -p gpurun_out
bash tools/gpu_kernel_variants.sh
STREAMS_LIST="*:1 *:2" bash tools/gpu_variants_streams.sh
timeout 300 python tools/e2e_timing.py > gpurun_out/e2e_timing.txt 2>&1; tail -8 gpurun_out/e2e_timing.txt
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_eval_cells|k_dseries" -c 2 -o gpurun_out/prof_r2h3 python tools/profile_run.py gpt-oss-120b 100 > gpurun_out/ncu_r2h3.log 2>&1; echo ncu_rc=$?
