# ncu full capture of the DP (C3, 296/launch) at a1f1eb6+revert, and the sort
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"dp_pass_kernel|seg_sort_kernel" -c 2 -o gpurun_out/r2_20_c3 -f \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_20_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r2_20_ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_20_launches_c3.csv \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_20_launch.log 2>&1; echo "launches rc=$?"
