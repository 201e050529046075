mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "concurrent or threads or host or golden_c3 or c4_64" > gpurun_out/r2_29_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_29_pytest.log
for st in 2 3 4; do for hc in 1 2 3 4; do python tools/e2e_probe.py 888 $st 3 $hc 2>&1 | head -2 | tr '\n' ' '; echo; done; done | tee gpurun_out/r2_29_e2e.log
python tools/e2e_probe.py 888 3 3 -1 2>&1 | head -2 | tr '\n' ' '
