mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_shard.py tests/test_gpu_envs.py -m "gpu and not slow" -q -x > gpurun_out/pytest_sparse.log 2>&1; echo "tests rc=$?" > gpurun_out/rc.txt
timeout 600 python tools/sparse_perf.py > gpurun_out/sparse_perf.txt 2>&1; echo "perf rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt; tail -3 gpurun_out/pytest_sparse.log; cat gpurun_out/sparse_perf.txt
