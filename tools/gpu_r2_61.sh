# non-aligned named barriers: synccheck, parity, A/B
mkdir -p gpurun_out/r2_61
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 20 \
    python tools/quick_bench.py C1:8 C3:2 C2:2 C4:4 > gpurun_out/r2_61/synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY" gpurun_out/r2_61/synccheck.log | head -3
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_61/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2_61/pytest.log
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_61/ab.log
