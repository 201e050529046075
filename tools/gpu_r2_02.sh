# fused DP pricing: focused parity first, then the whole GPU suite and a C3 bench line
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "dp_pricing or golden_c3 or golden_c1 or c4_subset" > gpurun_out/r2_02_pytest_focus.log 2>&1; echo "focus rc=$?"
tail -15 gpurun_out/r2_02_pytest_focus.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_02_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2_02_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_02_bench_c3.json 2> gpurun_out/r2_02_bench_c3.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_02_bench_c3.err
