# run-based need + interval candidate bins on the slice table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_16_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2_16_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "bin_intervals=0" 2>&1 | tee gpurun_out/r2_16_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" "bin_intervals=0" 2>&1 | tee gpurun_out/r2_16_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_table=1" 2>&1 | tee gpurun_out/r2_16_ab_c1.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_16_launches_c3.csv \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_16_launch.log 2>&1; echo "launches rc=$?"
