# windowed order search (n_clusters 9-10) + full GPU suite + sanitizers on the slice-table path
mkdir -p gpurun_out/r2_34
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_34/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_34/pytest.log
timeout 900 python -m pytest tests/test_order_search.py -q -k "more_than_eight" --durations=5 > gpurun_out/r2_34/order9.log 2>&1; tail -8 gpurun_out/r2_34/order9.log
for tool in racecheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 10 \
      python tools/quick_bench.py C1:8 C3:2 C4:4 > gpurun_out/r2_34/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/r2_34/sanitize_$tool.log | head -2
done
