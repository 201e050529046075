# full ncu capture of the slice-table DP pass (C3, 296/launch)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"dp_pass_kernel" -c 1 -o gpurun_out/r2_13_dp_c3 -f \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_13_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2_13_ncu.log
