timeout 600 python -m pytest tests/test_gpu_dense.py -x -q 2>&1 | tail -2
for mb in 0 24 48 96; do
  echo "== prefetch $mb MB"; RMB_PREFETCH_MB=$mb timeout 300 python tools/quick_perf.py 2>&1 | grep -E "b=10000|b=1000:|b=64"
done
