# final round-2 refresh (8-caller device-resident + e2e)
mkdir -p gpurun_out/r2_57
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_57/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2_57/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2_57/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_57/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_57/bench_c3.json 2> gpurun_out/r2_57/bench_c3.err; echo "c3 rc=$?"; head -c 700 gpurun_out/r2_57/bench_c3.json; echo
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_57/bench_ref_c3.json 2> gpurun_out/r2_57/bench_ref_c3.err; echo "ref rc=$?"; head -c 300 gpurun_out/r2_57/bench_ref_c3.json; echo
for c in C1 C2 C4; do timeout 900 python bench.py --config $c > gpurun_out/r2_57/bench_$c.json 2> gpurun_out/r2_57/bench_$c.err; echo "$c rc=$?"; head -c 200 gpurun_out/r2_57/bench_$c.json; echo; done
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 > gpurun_out/r2_57/bench_C5.json 2> gpurun_out/r2_57/bench_C5.err; echo "C5 rc=$?"; head -c 200 gpurun_out/r2_57/bench_C5.json; echo
timeout 900 python bench.py --config C4 --epoch --steps 5 --warmup 3 > gpurun_out/r2_57/bench_C4_epoch.json 2> gpurun_out/r2_57/bench_C4_epoch.err; echo "C4 epoch rc=$?"; head -c 200 gpurun_out/r2_57/bench_C4_epoch.json; echo
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"dp_pass_kernel|seg_sort_kernel|gtab_bins_kernel|rowexit_kernel" -c 4 -o gpurun_out/r2_57/c3 -f \
    python tools/quick_bench.py C3:296 > gpurun_out/r2_57/ncu.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/r2_57/ncu.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_57/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_57/launch.log 2>&1; echo "launches rc=$?"
