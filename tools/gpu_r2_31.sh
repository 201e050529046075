# drop-in latency (C++ dp_partition / plan_minibatches) + sanitizers on the slice-table path
mkdir -p gpurun_out/r2_31
timeout 600 ./build/dropin_latency 48 2>&1 | tee gpurun_out/r2_31/dropin_latency.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/quick_bench.py C1:8 C3:2 C2:2 C4:4 > gpurun_out/r2_31/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error" gpurun_out/r2_31/sanitize_$tool.log | head -4
done
QB_TUNE="slice_table=0" timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
      python tools/quick_bench.py C3:2 C4:4 > gpurun_out/r2_31/sanitize_racecheck_band.log 2>&1
echo "racecheck band rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY" gpurun_out/r2_31/sanitize_racecheck_band.log | head -3
