# compute-sanitizer on the sanitizer builds (600 s watchdog), the small
# workloads of tools/sanitize_check.py; full logs under gpurun_out/
mkdir -p gpurun_out
export FLOE_LIB=tools/libfloe_b200_sanitize.so
for tool in memcheck synccheck; do
  echo "--- $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 40 python tools/sanitize_check.py > gpurun_out/$tool.log 2>&1
  grep -E "workload ok|ERROR SUMMARY|Error|Traceback" gpurun_out/$tool.log | head -8
done
echo "--- racecheck (FLOE_RACECHECK build)"
FLOE_LIB=tools/libfloe_b200_racecheck.so timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all \
  --print-limit 40 python tools/sanitize_check.py > gpurun_out/racecheck.log 2>&1
grep -E "workload ok|RACECHECK SUMMARY|Traceback" gpurun_out/racecheck.log | head -8
