# Current-state snapshot: phase trace (layer + expert + steady state), batched layer (config 4/5), EP bench line.
timeout 600 python tools/exp_phases.py > gpurun_out/phases.txt 2>&1; echo phases rc=$?
timeout 900 python tools/bench_blayer.py > gpurun_out/blayer.jsonl 2> gpurun_out/blayer.err; echo blayer rc=$?
timeout 600 python bench.py --ep --steps 5 --warmup 3 > gpurun_out/ep.json 2> gpurun_out/ep.err; echo ep rc=$?
