# four accumulators per worker in the keyed far-far loop
mkdir -p gpurun_out/r2_48
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_48/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_48/pytest.log
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_48/ab.log
