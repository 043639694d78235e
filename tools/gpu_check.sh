# One-call GPU check: parity tests (twice), smoke, phase trace, bench, host repro.
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python tools/repro_host.py 2>&1 | tail -2
timeout 300 python tools/exp_phases.py 2>&1 | grep -E "t\[|first start|slowest" | head -30
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('LAYER us', d['ms_per_step']*1e3, 'tok/s', d['value'], 'frac', d['step_roofline']['frac'], 'EXPERT us', d['expert_ffn']['us_per_expert_token'], 'e2e', d['e2e']['value'])"
