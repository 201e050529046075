# sort CTA size by segment length (128 / 256 / 512 threads)
mkdir -p gpurun_out/r2_51
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_dropin.py -x -q > gpurun_out/r2_51/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_51/pytest.log
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_51/ab.log
