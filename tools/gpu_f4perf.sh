mkdir -p gpurun_out
timeout 900 python tools/f4_perf.py > gpurun_out/f4_perf.txt 2>&1; echo "rc=$?"; cat gpurun_out/f4_perf.txt | tail -30
