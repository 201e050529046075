# select_recomputation on the device + the full GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "recomputation or op_cost" > gpurun_out/r2_21_sel.log 2>&1; echo "sel rc=$?"; tail -5 gpurun_out/r2_21_sel.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_21_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_21_pytest.log
