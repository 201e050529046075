timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"band_run_kernel|dp_pass_kernel" -c 2 -o gpurun_out/r2_04_priced_c3 -f \
    python tools/quick_bench.py C3:148 > gpurun_out/r2_04_ncu.log 2>&1; echo "ncu rc=$?"
QB_TUNE="dp_pricing=0" timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"band_run_kernel|dp_pass_kernel" -c 2 -o gpurun_out/r2_04_band_c3 -f \
    python tools/quick_bench.py C3:148 > gpurun_out/r2_04_ncu_band.log 2>&1; echo "ncu band rc=$?"
