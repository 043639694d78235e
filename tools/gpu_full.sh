# Round evidence: tests, smoke, bench (with CPU baseline), reference arm, ncu launch list + full capture, config-3 decode.
set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -2 gpurun_out/bench_r01.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -2 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 66 -c 1 -o gpurun_out/prof_r01 python tools/prof_layer.py --steps 4 > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
rm -f gpurun_out/config3.jsonl; timeout 600 python tools/bench_offload.py --out gpurun_out/config3.jsonl > gpurun_out/off32.log 2>&1; echo config3 rc=$?; cat gpurun_out/config3.jsonl
