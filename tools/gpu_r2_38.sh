# cp.async unit fill in the DP producer
mkdir -p gpurun_out/r2_38
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_38/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_38/pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_38/ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" 2>&1 | tee gpurun_out/r2_38/ab_c4.log
for m in 1 296; do echo "== DP_M=$m"; DP_M=$m PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tail -13; done | tee gpurun_out/r2_38/trace.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 10 python tools/quick_bench.py C1:8 C3:2 C4:4 > gpurun_out/r2_38/racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY" gpurun_out/r2_38/racecheck.log
