# DP phase sums (chain path vs worker path per block) for C3 / C4
mkdir -p gpurun_out/r2_47
for c in C3 C4; do for m in 1 296; do echo "== $c DP_M=$m"; DP_M=$m PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py $c 2>&1 | tail -24; done; done | tee gpurun_out/r2_47/trace.log
