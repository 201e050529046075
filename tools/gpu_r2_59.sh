# C5 line (one caller for very long mini-batches)
mkdir -p gpurun_out/r2_59
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/r2_59/bench_C5.json 2> gpurun_out/r2_59/bench_C5.err; echo "C5 rc=$?"; head -c 400 gpurun_out/r2_59/bench_C5.json; echo
