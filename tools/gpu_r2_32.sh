# T5 per-kind slice-time tables for cost pass B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "kind_tables or c2 or golden or replicas_and_capped or c5 or exact" > gpurun_out/r2_32_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_32_pytest.log
timeout 600 python tools/ab_bench.py C2 192 "slice_table=1" "kind_tables=0" 2>&1 | tee gpurun_out/r2_32_ab_c2.log
