# TMA-fed slice table: focused parity, A/B against the band, per-block trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "slice_table or golden or c4 or slice_reuse or nan_interval or dp_pricing" > gpurun_out/r2_09_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_09_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_09_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_09_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_09_ab_c1.log
PP_TRACE=1 python -c "from paper_2311_10418_b200 import build as b; b.build()" > /dev/null 2>&1
for c in C3 C4; do echo "== $c gtab"; PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py $c; done 2>&1 | tee gpurun_out/r2_09_trace.log
