# fix: partial-triangle prefetch start
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_18_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_18_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_18_ab_c3.log
for hc in 2 3 4; do for st in 3 4; do timeout 300 python tools/e2e_probe.py 888 $st 5 $hc 2>&1 | head -3; done; done | tee gpurun_out/r2_18_e2e.log
