# One-call GPU check: parity tests, smoke, phase trace, bench.
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
timeout 300 python tools/exp_phases.py 2>&1 | head -24
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; python -c "
import json; d=json.load(open('gpurun_out/bench.json')); print('LAYER us', d['ms_per_step']*1e3, 'tok/s', d['value'], 'frac', d['step_roofline']['frac'], 'EXPERT us', d['expert_ffn']['us_per_expert_token'], 'e2e', d['e2e']['value'])"
