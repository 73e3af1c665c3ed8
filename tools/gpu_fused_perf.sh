mkdir -p gpurun_out
timeout 600 python tools/check_sharded_c2.py > gpurun_out/fused_perf.txt 2>&1; echo "rc=$?"; cat gpurun_out/fused_perf.txt | tail -5
