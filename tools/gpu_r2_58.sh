# the chain reduces far-far chunks from the back after its triangle (HELP)
mkdir -p gpurun_out/r2_58
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_dropin.py -x -q > gpurun_out/r2_58/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_58/pytest.log
for c in "C3 296" "C4 512" "C1 2048"; do timeout 600 python tools/ab_bench.py $c "slice_table=1" 2>&1; done | tee gpurun_out/r2_58/ab.log
for c in C3 C4; do echo "== $c DP_M=296"; DP_M=296 PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py $c 2>&1 | tail -24; done | tee gpurun_out/r2_58/trace.log
