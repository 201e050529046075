timeout 600 python tools/ab_bench.py C3 296 "dp_pricing=1" "dp_pricing=0" "dp_pricing=0,compact_band=1" "dp_pricing=1,streams=3" "dp_pricing=0,streams=3" "dp_pricing=0,compact_band=1,streams=3" 2>&1 | tee gpurun_out/r2_03_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "dp_pricing=1" "dp_pricing=0" "dp_pricing=0,compact_band=1" 2>&1 | tee gpurun_out/r2_03_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "dp_pricing=1" "dp_pricing=0" "dp_pricing=0,compact_band=1" 2>&1 | tee gpurun_out/r2_03_ab_c1.log
