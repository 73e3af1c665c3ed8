mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dense.py -q -x -k "cluster" > gpurun_out/pytest_cluster.log 2>&1; echo "cluster tests rc=$?"; tail -30 gpurun_out/pytest_cluster.log
timeout 300 python tools/ab_tma.py 3,2,1 > gpurun_out/ab_small.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_small.txt
