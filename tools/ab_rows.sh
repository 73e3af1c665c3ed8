for v in v0 v1 default; do
  if [ $v = default ]; then L=""; else L="RMB_LIB_PATH=exp/librmb_$v.so"; fi
  echo "== $v"; env $L timeout 300 python tools/quick_perf.py 2>&1 | grep -E "b=10000|b=1000:"
  echo "== $v warp"; env $L RMB_DENSE_ROWS=0 timeout 300 python tools/quick_perf.py 2>&1 | grep -E "b=10000|b=1000:"
done
