# redesigned DP kernel (redundant serial chain, on-the-fly near-far, units, direct G reads)
mkdir -p gpurun_out
timeout 600 python -c "
import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_10_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2_10_smoke.log
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2_10_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2_10_pytest.log
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_10_ab_c3.log
timeout 600 python tools/ab_bench.py C4 512 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_10_ab_c4.log
timeout 600 python tools/ab_bench.py C1 2048 "slice_table=1" "slice_table=0" 2>&1 | tee gpurun_out/r2_10_ab_c1.log
timeout 600 python tools/ab_bench.py C2 192 "slice_table=1" 2>&1 | tee gpurun_out/r2_10_ab_c2.log
PP_TRACE=1 python -c "from paper_2311_10418_b200 import build as b; b.build()" > /dev/null 2>&1
for t in "slice_table=1" "slice_table=0"; do for c in C3 C4; do echo "== $c $t"; QB_TUNE=$t PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py $c; done; done 2>&1 | tee gpurun_out/r2_10_trace.log
