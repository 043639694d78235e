timeout 900 python -m pytest tests/test_gpu_offload_timeline.py tests/test_gpu_offload.py tests/test_gpu_parity_bench.py -x -q 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('BENCH tok/s', d['value'], 'us/layer', d['layer']['us_per_layer'], 'frac', d['roofline']['frac']); print(json.dumps(d.get('offload')))"
