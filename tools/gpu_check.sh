# Full GPU check: smoke, -m gpu tests, default bench, launch list, one ncu --set full capture.
# usage: bash tools/gpu_check.sh TAG
TAG=${1:-r1}
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/lscpu.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_$TAG.json
timeout 300 python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/bench_small_$TAG.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-bsweep --no-e2e --no-cpu --no-other > gpurun_out/ncu_launch_$TAG.log 2>&1; echo launches rc=$?
timeout 120 python tools/prof_dense.py 1000 20 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dense_(tma|solver)" -c 1 -o gpurun_out/dense_b1000_$TAG python tools/prof_dense.py 1000 20 > gpurun_out/ncu_full_$TAG.log 2>&1; echo full rc=$?
