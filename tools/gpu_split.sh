mkdir -p gpurun_out
for k in 1 2 3 4; do
  timeout 600 python bench.py --no-cpu-baseline --split $k > gpurun_out/split_$k.json 2>gpurun_out/split_$k.err
  python -c "
import json; d=json.load(open('gpurun_out/split_$k.json'))
print('split $k ms/step', round(d['ms_per_step'],3), 'e2e', round(d['search_wall_ms']['e2e'],3), 'seq', round(d['search_wall_ms']['per_model_sequential_device'],3), 'launches', d['gpu_launches'])" || tail -3 gpurun_out/split_$k.err
done
