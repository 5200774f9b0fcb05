# diagnostics: K5a merge counts (LC_COUNT_MERGES build in variants/diag/count.so) and the e2e host phases
mkdir -p gpurun_out
for m in gpt-oss-120b deepseek-v3; do
  LC_B200_LIB=variants/diag/count.so timeout 300 python tools/profile_run.py $m 100 2>&1 | grep -E "merges|candidates" | tail -3
done
LC_HOST_TIMING=1 timeout 300 python tools/e2e_timing.py > gpurun_out/e2e_timing3.txt 2>&1; tail -8 gpurun_out/e2e_timing3.txt
