# Round evidence: bench (full line), reference arm, ncu launch list, one ncu --set full capture
# of the decode kernel (32 layers), steady-state phase trace.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/bench_ev.json 2> gpurun_out/bench_ev.err; tail -2 gpurun_out/bench_ev.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_ev.json 2> gpurun_out/bench_ref_ev.err; cat gpurun_out/bench_ref_ev.json | head -c 400
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:decode -c 200 --csv --log-file gpurun_out/launches_ev.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-offload > /dev/null 2>&1; echo ncu_launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_ev python tools/prof_multi.py 32 > gpurun_out/ncu_full_ev.log 2>&1; echo ncu_full rc=$?
timeout 300 python tools/trace_multi.py > gpurun_out/trace_ev.txt 2>&1; echo trace rc=$?
