# host-buffer pipeline: parts planned one after another, copies on two copy streams
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_25_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_25_pytest.log
for hc in 0 2 4 6 8 -2; do python tools/e2e_probe.py 888 3 3 $hc 2>&1 | head -2; done | tee gpurun_out/r2_25_e2e.log
