#!/bin/bash
# One gpurun call: GPU tests (fast set, then the full-size set) + a short bench line.
#   gpurun --timeout 2400 -- bash tools/gpu_check.sh [pytest -k expr]
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt 2>&1; free -g > gpurun_out/free.txt
K=${1:-}
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x ${K:+-k "$K"} > gpurun_out/pytest_fast.log 2>&1
echo "fast rc=$?" >> gpurun_out/rc.txt
timeout 1800 python -m pytest tests -m "gpu and slow" -q --durations=0 ${K:+-k "$K"} > gpurun_out/pytest_slow.log 2>&1
echo "slow rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-other --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/rc.txt
tail -3 gpurun_out/pytest_fast.log gpurun_out/pytest_slow.log; cat gpurun_out/rc.txt
