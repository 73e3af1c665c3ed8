mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -q > gpurun_out/pytest_shard.log 2>&1; echo "shard rc=$?"; tail -3 gpurun_out/pytest_shard.log
