# per-kernel times (ncu launch list, one GPT-OSS-120B + one DeepSeek-V3 batch of 100 config-5 searches)
# for every variants/*.so:  bash tools/gpu_kernel_variants.sh
mkdir -p gpurun_out
for so in variants/*.so; do
  n=$(basename $so .so)
  for m in gpt-oss-120b deepseek-v3; do
    LC_B200_LIB=$so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/kt_${n}_${m}.csv python tools/profile_run.py $m 100 > /dev/null 2>&1
  done
  python tools/kernel_times.py gpurun_out/kt_${n}_gpt-oss-120b.csv gpurun_out/kt_${n}_deepseek-v3.csv
done
