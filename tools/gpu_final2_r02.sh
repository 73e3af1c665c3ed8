mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu -rf > gpurun_out/gpu_all_final3.txt 2>&1; echo "gpu tests rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/gpu_all_final3.txt | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc=$?"
