mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/pytest_fast.log 2>&1; echo "fast rc=$?" > gpurun_out/rc.txt
timeout 1200 python -m pytest tests -m "gpu and slow" -q --durations=5 > gpurun_out/pytest_slow.log 2>&1; echo "slow rc=$?" >> gpurun_out/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt; tail -3 gpurun_out/pytest_fast.log; tail -8 gpurun_out/pytest_slow.log; tail -2 gpurun_out/smoke.log
