mkdir -p gpurun_out/r2_35
timeout 900 python -m pytest tests/test_order_search.py -x -q > gpurun_out/r2_35/order.log 2>&1; echo "order rc=$?"; tail -15 gpurun_out/r2_35/order.log
