# int32 slice-table bases + shuffled column bases in the DP worker loop
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_14_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_14_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_14_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" 2>&1 | tee gpurun_out/r2_14_ab_c4.log
