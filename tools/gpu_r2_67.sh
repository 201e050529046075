# final validation at HEAD: smoke, every -m gpu test, C3 + C4 bench lines
mkdir -p gpurun_out/r2_67
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_67/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_67/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_67/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_67/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_67/bench_c3.json 2> gpurun_out/r2_67/bench_c3.err; echo "c3 rc=$?"; head -c 300 gpurun_out/r2_67/bench_c3.json; echo
timeout 900 python bench.py --config C4 > gpurun_out/r2_67/bench_C4.json 2> gpurun_out/r2_67/bench_C4.err; echo "C4 rc=$?"; head -c 300 gpurun_out/r2_67/bench_C4.json; echo
