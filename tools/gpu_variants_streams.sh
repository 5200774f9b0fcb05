# time every variants/*.so with the config5 bench at several --streams settings
#   STREAMS_LIST="*:1 *:2" bash tools/gpu_variants_streams.sh
mkdir -p gpurun_out
for so in variants/*.so; do
  n=$(basename $so .so)
  for st in ${STREAMS_LIST:-*:1 *:2}; do
    LC_B200_LIB=$so timeout 600 python bench.py --no-cpu-baseline --north-star none --steps 30 --streams "$st" > gpurun_out/var_${n}.json 2>/dev/null
    python -c "
import json,sys; d=json.load(open('gpurun_out/var_$n.json'))
print('$n', '$st', 'ms/step', round(d['ms_per_step'],3), 'e2e', round(d['search_wall_ms']['e2e'],3), 'seq', round(d['search_wall_ms']['per_model_sequential_device'],3), {k: round(v,3) for k,v in d['roofline']['kernel_ms'].items()})" || echo "$n failed"
  done
done
