#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (SURVEY §4 layer 3). Logs in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 9 \
      --print-limit 200 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | head -3
  grep -E "Device Frame" gpurun_out/sanitize_$tool.log | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | head -8
done
