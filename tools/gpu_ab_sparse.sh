mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_envs.py tests/test_gpu_shard.py -q -x -m "gpu and not slow" > gpurun_out/pytest_sparse.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pytest_sparse.log
timeout 900 python tools/ab_sparse.py run > gpurun_out/ab_sparse.txt 2>&1; echo "ab rc=$?"
cat gpurun_out/ab_sparse.txt
