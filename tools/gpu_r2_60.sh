# sanitizers on the round-2 end state (producer-less slice-table DP, 7-bit sort, prefix outputs)
mkdir -p gpurun_out/r2_60
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/quick_bench.py C1:8 C3:2 C2:2 C4:4 > gpurun_out/r2_60/$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK SUMMARY|Hazard|barrier" gpurun_out/r2_60/$tool.log | head -5
done
