mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/gpu_all.txt 2>&1; echo "gpu tests rc=$?"; grep -E "FAILED|ERROR|passed|failed" gpurun_out/gpu_all.txt | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
