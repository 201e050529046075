# round-end style validation at HEAD: smoke, full GPU suite, bench C3 (+ launch list)
mkdir -p gpurun_out/r2_36
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_36/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_36/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_36/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_36/pytest.log
timeout 900 python bench.py > gpurun_out/r2_36/bench_c3.json 2> gpurun_out/r2_36/bench_c3.err; echo "bench rc=$?"; head -c 700 gpurun_out/r2_36/bench_c3.json; echo
