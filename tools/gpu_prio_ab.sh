# stream-priority A/B on the config5 bench (kernel-only numbers) and the north-star sweep
mkdir -p gpurun_out
for pr in none auto none auto; do
  for st in "*:1" "*:2"; do
    timeout 600 python bench.py --no-cpu-baseline --steps 30 --priority $pr --streams "$st" > gpurun_out/prio.json 2>gpurun_out/prio.err
    python -c "
import json; d=json.load(open('gpurun_out/prio.json'))
print('$pr', '$st', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['search_wall_ms']['e2e'],3), 'ns', round(d['north_star']['ms_per_step'],3), round(d['north_star']['e2e_ms_per_step'],3))" || tail -3 gpurun_out/prio.err
  done
done
