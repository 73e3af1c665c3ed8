for v in default st28672 st24576; do
  if [ $v = default ]; then L=""; else L="RMB_LIB_PATH=exp/librmb_$v.so"; fi
  echo "== $v"; env $L timeout 200 python tools/ab_tma.py 10000,1000,250,64 2>&1 | grep "^tma"
done
