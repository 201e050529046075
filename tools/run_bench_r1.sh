#!/bin/bash
# bench line + reference arm + launch list (run under gpurun from the repo root)
OUT=gpurun_out
nproc > $OUT/nproc.txt; lscpu > $OUT/lscpu.txt 2>&1
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 4 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "ncu rc=$?"
