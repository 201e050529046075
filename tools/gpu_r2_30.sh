# bench lines at HEAD: C3 (default), reference arm, C1 / C2 / C4 / C5 configs, C4 epoch (1 GPU)
mkdir -p gpurun_out/r2_30
timeout 900 python bench.py > gpurun_out/r2_30/bench_c3.json 2> gpurun_out/r2_30/bench_c3.err; echo "c3 rc=$?"; head -c 600 gpurun_out/r2_30/bench_c3.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_30/bench_ref_c3.json 2> gpurun_out/r2_30/bench_ref_c3.err; echo "ref rc=$?"; head -c 400 gpurun_out/r2_30/bench_ref_c3.json; echo
for c in C1 C2 C4; do timeout 900 python bench.py --config $c > gpurun_out/r2_30/bench_$c.json 2> gpurun_out/r2_30/bench_$c.err; echo "$c rc=$?"; head -c 300 gpurun_out/r2_30/bench_$c.json; echo; done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/r2_30/bench_C5.json 2> gpurun_out/r2_30/bench_C5.err; echo "C5 rc=$?"; head -c 300 gpurun_out/r2_30/bench_C5.json; echo
timeout 900 python bench.py --config C4 --epoch --steps 5 --warmup 3 > gpurun_out/r2_30/bench_C4_epoch.json 2> gpurun_out/r2_30/bench_C4_epoch.err; echo "C4 epoch rc=$?"; head -c 400 gpurun_out/r2_30/bench_C4_epoch.json; echo
