# HEAD (slice table) C3: launch list + full ncu capture of the DP and slice-table kernels, DP trace
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_12_launches_c3.csv \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_12_launch.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"dp_pass_kernel|gtab|seg_sort" -c 6 -o gpurun_out/r2_12_full_c3 -f \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_12_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2_12_ncu.log
PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tee gpurun_out/r2_12_trace.log | tail -40
