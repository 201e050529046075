# e2e sweep at 1081101: streams x host_chunks, and a trace of the default
mkdir -p gpurun_out/r2_44
for s in 3 4 5 6; do for h in 0 2; do timeout 300 python tools/e2e_probe.py 888 $s 5 $h 2>&1 | grep -E "streams|host call|device call" | tr '\n' ' '; echo; done; done | tee gpurun_out/r2_44/sweep.log
timeout 300 python tools/e2e_probe.py 888 3 5 0 2>&1 | tail -6 | tee gpurun_out/r2_44/probe3.log
PP_E2E_TRACE=1 timeout 300 python tools/e2e_probe.py 888 3 2 0 > gpurun_out/r2_44/trace3.log 2>&1
PP_E2E_TRACE=1 timeout 300 python tools/e2e_probe.py 888 4 2 0 > gpurun_out/r2_44/trace4.log 2>&1
