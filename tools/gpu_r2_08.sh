# DP anatomy: per-block phase stamps (trace build) and one ncu --set full capture per DP variant
mkdir -p gpurun_out
for t in "slice_table=0" "slice_table=1"; do
  for c in C3 C4; do
    echo "== $c $t"; QB_TUNE=$t PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py $c
  done
done 2>&1 | tee gpurun_out/r2_08_trace.log
QB_TUNE="slice_table=0" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dp_pass_kernel" -c 1 -o gpurun_out/r2_08_dp_band -f python tools/quick_bench.py C3:148 > gpurun_out/r2_08_ncu_band.log 2>&1; echo "ncu rc=$?"
QB_TUNE="slice_table=1" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dp_pass_kernel" -c 1 -o gpurun_out/r2_08_dp_gtab -f python tools/quick_bench.py C3:148 > gpurun_out/r2_08_ncu_gtab.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
