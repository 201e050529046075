# broadcast triangle (one fold + one shuffle round trip per row)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_24_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_24_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_24_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" 2>&1 | tee gpurun_out/r2_24_ab_c4.log
timeout 600 python tools/ab_bench.py C2 192 "slice_table=1" 2>&1 | tee gpurun_out/r2_24_ab_c2.log
for m in 1 296; do echo "== DP_M=$m"; DP_M=$m PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tail -11; done | tee gpurun_out/r2_24_trace.log
