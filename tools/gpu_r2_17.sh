# PTX lexicographic select on the chain's descending folds + bins test fix
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_17_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_17_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_17_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" 2>&1 | tee gpurun_out/r2_17_ab_c4.log
PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tee gpurun_out/r2_17_trace.log | tail -12
