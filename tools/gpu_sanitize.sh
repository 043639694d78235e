# compute-sanitizer on the sanitizer build (600 s watchdog), the small workloads of tools/sanitize_check.py
export FLOE_LIB=tools/libfloe_b200_sanitize.so
for tool in memcheck racecheck synccheck; do
  echo "--- $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_check.py 2>&1 | grep -E "workload ok|ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Hazard|error" | head -20
done
