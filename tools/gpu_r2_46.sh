# prioritised worker streams on the host path (later parts first)
mkdir -p gpurun_out/r2_46
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "pinned or order_output or host or thread" > gpurun_out/r2_46/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_46/pytest.log
for r in 1 2; do
for a in "3 5 0" "4 5 0"; do timeout 300 python tools/e2e_probe.py 888 $a 2>&1 | grep -E "streams|host call" | tr '\n' ' '; echo; done
for a in "3 5 0"; do PP_HOST_NO_PRIO=1 timeout 300 python tools/e2e_probe.py 888 $a 2>&1 | grep -E "streams|host call" | tr '\n' ' '; echo " (no prio)"; done
done | tee gpurun_out/r2_46/sweep.log
PP_E2E_TRACE=1 timeout 300 python tools/e2e_probe.py 888 3 2 0 > gpurun_out/r2_46/trace3.log 2>&1
