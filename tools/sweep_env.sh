# Sweep runtime knobs of the fused kernel: layer us (32-layer decode, steady state) per setting.
# usage: bash tools/sweep_env.sh "FLOE_NSC=8" "FLOE_NSC=12 FLOE_EARLY=4" ...
for cfg in "$@"; do
  r=$(env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-offload 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('us/layer %.2f frac %.3f' % (d['layer']['us_per_layer'], d['roofline']['frac']))")
  echo "$cfg -> $r"
done
