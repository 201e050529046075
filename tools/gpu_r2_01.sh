set -x
nproc > gpurun_out/r2_01_nproc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_01_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2_01_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_01_bench_c3.json 2> gpurun_out/r2_01_bench_c3.err; echo "bench rc=$?"
timeout 900 python bench.py --config C4 --epoch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_01_bench_c4e.json 2> gpurun_out/r2_01_bench_c4e.err; echo "bench c4 rc=$?"
tail -3 gpurun_out/r2_01_bench_c4e.err
