# re-validation after container restore: whole GPU suite at HEAD, C3 bench line, C4 epoch line, slice-table A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_07_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_07_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_07_bench_c3.json 2> gpurun_out/r2_07_bench_c3.err; echo "bench rc=$?"; tail -3 gpurun_out/r2_07_bench_c3.err
timeout 600 python bench.py --config C4 --epoch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_07_bench_c4e.json 2> gpurun_out/r2_07_bench_c4e.err; echo "bench c4 rc=$?"; tail -3 gpurun_out/r2_07_bench_c4e.err
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "slice_table=0" "slice_table=0,dp_pricing=1" 2>&1 | tee gpurun_out/r2_07_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_07_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_07_ab_c1.log
