# One-call GPU check: bench on both paths + ncu launch list of the default path.
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; tail -3 gpurun_out/bench_fused.err; cat gpurun_out/bench_fused.json
FLOE_GPU_PATH=split timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_split.json 2> gpurun_out/bench_split.err; tail -3 gpurun_out/bench_split.err; cat gpurun_out/bench_split.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
