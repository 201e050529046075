# chain timing: alone vs with workers, 1 CTA vs 2 CTAs per SM
mkdir -p gpurun_out
for m in 1 296; do for f in 0 1; do echo "== DP_M=$m DP_FLAGS=$f"; DP_M=$m DP_FLAGS=$f PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tail -11; done; done | tee gpurun_out/r2_23_trace.log
