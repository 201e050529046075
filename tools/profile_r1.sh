#!/bin/bash
# Round-1 profiling recipe (run under gpurun from the repo root).
set -x
OUT=gpurun_out
timeout 600 python tools/quick_bench.py C1:1 C1:64 C2:1 C2:16 C3:1 C3:8 C3:32 C4:64 C4:512 > $OUT/quick.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"block_kernel|dp_pass_kernel" -s 4 -c 4 -o $OUT/prof_c3 -f \
    python tools/quick_bench.py C3:8 > $OUT/ncu_full.log 2>&1
timeout 600 python tools/quick_bench.py C5:1 > $OUT/quick_c5.log 2>&1
echo done
