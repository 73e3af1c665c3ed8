mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_async.py -q -m gpu > gpurun_out/async_tests.txt 2>&1; echo "async rc=$?"; grep -E "FAILED|passed|failed|Error|error" gpurun_out/async_tests.txt | head -30
