# vectorised small_copy, host path default 2 x streams workers
mkdir -p gpurun_out/r2_45
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "pinned or order_output or host or thread" > gpurun_out/r2_45/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_45/pytest.log
for a in "3 5 0" "3 5 1" "4 5 0" "2 5 0"; do timeout 300 python tools/e2e_probe.py 888 $a 2>&1 | grep -E "streams|host call|device call" | tr '\n' ' '; echo; done | tee gpurun_out/r2_45/sweep.log
PP_E2E_TRACE=1 timeout 300 python tools/e2e_probe.py 888 3 2 0 > gpurun_out/r2_45/trace3.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_45/bench_c3.json 2> gpurun_out/r2_45/bench_c3.err; echo "c3 rc=$?"; head -c 1000 gpurun_out/r2_45/bench_c3.json; echo
