#!/bin/bash
# bench line (+ reference arm) + launch list + full ncu capture of the top kernels
# (run under gpurun from the repo root).  Usage: bash tools/run_bench_r1.sh TAG
TAG=${1:-run}
OUT=gpurun_out
nproc > $OUT/nproc.txt
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 4 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --streams 1 --per-gpu 296 > $OUT/ncu_bench_$TAG.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"band_run_kernel|band3_kernel|band_kernel|block_kernel|dp_pass_kernel" -s 6 -c 4 -o $OUT/prof_$TAG -f \
    python tools/quick_bench.py C3:148 > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
