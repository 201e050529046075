mkdir -p gpurun_out/r2_37
timeout 600 python tools/ab_bench.py C3 296 "slice_table=1" 2>&1 | tee gpurun_out/r2_37/ab_c3.log
for m in 1 296; do echo "== DP_M=$m"; DP_M=$m PIPEPLAN_B200_LIB=build/trace/libpipeplan_b200_trace.so timeout 300 python tools/dp_trace.py C3 2>&1 | tail -13; done | tee gpurun_out/r2_37/trace.log
timeout 900 ./build/tsan/acceptance_dropin > gpurun_out/r2_37/tsan_acceptance.log 2>&1; echo "tsan acceptance rc=$?"; grep -c "WARNING: ThreadSanitizer" gpurun_out/r2_37/tsan_acceptance.log; tail -3 gpurun_out/r2_37/tsan_acceptance.log
timeout 900 ./build/tsan/epoch_dropin /tmp/ept > gpurun_out/r2_37/tsan_epoch.log 2>&1; echo "tsan epoch rc=$?"; grep -c "WARNING: ThreadSanitizer" gpurun_out/r2_37/tsan_epoch.log; tail -3 gpurun_out/r2_37/tsan_epoch.log
