# full ncu capture of selected kernels: bash tools/gpu_ncu_k.sh <tag> <regex> <model> <count>
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$2" -s ${5:-0} -c $4 -o gpurun_out/prof_$1 python tools/profile_run.py $3 100 > gpurun_out/ncu_$1.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_$1.log
