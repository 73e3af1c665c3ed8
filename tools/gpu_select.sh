mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_select.py -q -m gpu > gpurun_out/select_tests.txt 2>&1; echo "select rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/select_tests.txt | head -40
