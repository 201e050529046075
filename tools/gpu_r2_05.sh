timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_05_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_05_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "dp_pricing=0" "dp_pricing=1" 2>&1 | tee gpurun_out/r2_05_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "dp_pricing=0" 2>&1 | tee gpurun_out/r2_05_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "dp_pricing=0" 2>&1 | tee gpurun_out/r2_05_ab_c1.log
