# Layer/expert step time under a few environment settings (one short bench each).
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/sweep.json 2> /dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); print('$cfg', 'LAYER us', round(d['ms_per_step']*1e3,2), 'EXPERT us', d['expert_ffn']['us_per_expert_token'])"
done
