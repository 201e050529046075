# kind tables (T5 pass B) + named-barrier unit hand-off: parity, timing, sanitizers
mkdir -p gpurun_out/r2_33
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_33/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_33/pytest.log
timeout 600 python tools/ab_bench.py C2 192 "slice_table=1" "kind_tables=0" 2>&1 | tee gpurun_out/r2_33/ab_c2.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_33/ab_c3.log
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 \
      python tools/quick_bench.py C1:8 C3:2 C2:2 C4:4 > gpurun_out/r2_33/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r2_33/sanitize_$tool.log | head -2
done
