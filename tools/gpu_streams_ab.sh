mkdir -p gpurun_out
for st in "*:1" "gpt-oss-120b:2,qwen3-32b:2" "gpt-oss-120b:3,qwen3-32b:3" "*:2" "gpt-oss-120b:3,deepseek-v3:2,qwen3-32b:3"; do
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --streams "$st" > gpurun_out/st.json 2>gpurun_out/st.err
  python -c "
import json; d=json.load(open('gpurun_out/st.json'))
print('$st', 'ms', round(d['ms_per_step'],3), 'e2e', round(d['search_wall_ms']['e2e'],3), 'seq', round(d['search_wall_ms']['per_model_sequential_device'],3), 'ns', round(d['north_star']['ms_per_step'],3), round(d['north_star']['e2e_ms_per_step'],3))" || tail -3 gpurun_out/st.err
done
