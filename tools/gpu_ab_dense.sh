mkdir -p gpurun_out
timeout 300 python tools/ab_tma.py 10000,1000,64 > gpurun_out/ab_la2.txt 2>&1; echo "ab rc=$?"; grep "^tma" gpurun_out/ab_la2.txt
timeout 300 python tools/check_sharded_c2.py > gpurun_out/fused_perf_la2.txt 2>&1; echo "fused rc=$?"; tail -2 gpurun_out/fused_perf_la2.txt
