# need_runs at 32 warps for long segments; then the full GPU suite + smoke at HEAD
mkdir -p gpurun_out/r2_64
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_64/ab.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_64/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_64/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_64/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_64/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_64/bench_c3.json 2> gpurun_out/r2_64/bench_c3.err; echo "c3 rc=$?"; head -c 300 gpurun_out/r2_64/bench_c3.json; echo
