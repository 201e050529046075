# keyed counts (count|column in one int) in the slice-table far-far loop
mkdir -p gpurun_out/r2_43
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_43/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_43/pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_43/ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" 2>&1 | tee gpurun_out/r2_43/ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_table=1" 2>&1 | tee gpurun_out/r2_43/ab_c1.log
for m in 1 296; do echo "== DP_M=$m"; DP_M=$m PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tail -13; done | tee gpurun_out/r2_43/trace.log
timeout 900 python bench.py > gpurun_out/r2_43/bench_c3.json 2> gpurun_out/r2_43/bench_c3.err; echo "c3 rc=$?"; head -c 1200 gpurun_out/r2_43/bench_c3.json; echo
