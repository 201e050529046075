# 7-bit ranked radix passes (match_any) for one-word sort keys
mkdir -p gpurun_out/r2_50
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_50/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_50/pytest.log
for c in "C3 296" "C4 512" "C1 2048" "C2 192"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_50/ab.log
