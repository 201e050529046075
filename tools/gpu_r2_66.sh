# second pairing level of worker partials (chain folds two)
mkdir -p gpurun_out/r2_66
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_66/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_66/pytest.log
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_66/ab.log
