for k in 1 2 3 4 6 8 12; do
  echo "== IPW=$k"; RMB_DENSE_IPW=$k timeout 300 python tools/quick_perf.py 1000,64,250,2000 x 2>&1 | grep -E "b="
done
