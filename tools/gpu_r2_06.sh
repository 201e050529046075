timeout 600 python tools/ab_bench.py C4 512 "slice_reuse=1" "slice_reuse=0" "slice_reuse=1,band_trunc=0" 2>&1 | tee gpurun_out/r2_06_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_reuse=1" "slice_reuse=0" 2>&1 | tee gpurun_out/r2_06_ab_c1.log
timeout 600 python tools/ab_bench.py C2 192 "slice_reuse=1" 2>&1 | tee gpurun_out/r2_06_ab_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_run_kernel|dp_pass_kernel" -c 2 -o gpurun_out/r2_06_c4 -f python tools/quick_bench.py C4:512 > gpurun_out/r2_06_ncu.log 2>&1; echo "ncu rc=$?"
