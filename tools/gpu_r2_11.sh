# re-entry validation of HEAD: smoke, full GPU suite, C3 bench, A/B slice table
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_11_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2_11_smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_11_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_11_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_11_bench_c3.json 2> gpurun_out/r2_11_bench_c3.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2_11_bench_c3.json
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_11_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_11_ab_c4.log
