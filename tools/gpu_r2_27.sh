# small transfers of the planning path through mapped pinned memory + kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_27_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_27_pytest.log
for hc in 0 2 4 6 -1 -2; do python tools/e2e_probe.py 888 3 3 $hc 2>&1 | head -2; done | tee gpurun_out/r2_27_e2e.log
python tools/e2e_probe.py 888 3 3 6 2>&1 | tail -6
