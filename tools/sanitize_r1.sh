#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over a small planning workload
OUT=gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/quick_bench.py C1:8 C3:2 C2:2 > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|Error|error" $OUT/sanitize_$tool.log | head -5
done
