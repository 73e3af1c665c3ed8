mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q -x -k "fused" > gpurun_out/pytest_fused.log 2>&1; echo "fused rc=$?"
tail -30 gpurun_out/pytest_fused.log
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_dense.py -q -x -m "gpu and not slow" > gpurun_out/pytest_dense_shard.log 2>&1; echo "all rc=$?"
tail -3 gpurun_out/pytest_dense_shard.log
