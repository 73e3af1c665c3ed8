for v in default bar1; do
  if [ $v = default ]; then L=""; else L="RMB_LIB_PATH=exp/librmb_$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/quick_perf.py 2>&1 | grep -E "b="
done
RMB_LIB_PATH=exp/librmb_bar1.so timeout 600 python -m pytest tests/test_gpu_dense.py tests/test_gpu_sparse.py -x -q 2>&1 | tail -2
