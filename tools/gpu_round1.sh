set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_r1.json
timeout 300 python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu > gpurun_out/bench_small.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 120 python tools/prof_dense.py 1000 20 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_solver -c 1 -o gpurun_out/dense_b1000_r1 python tools/prof_dense.py 1000 20 > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
