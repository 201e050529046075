# full GPU suite after the DP chain / worker / slice-table changes
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_19_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_19_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_19_ab_c3.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_19_bench_c3.json 2> gpurun_out/r2_19_bench_c3.err; echo "bench rc=$?"; head -c 1200 gpurun_out/r2_19_bench_c3.json; tail -3 gpurun_out/r2_19_bench_c3.err
