for v in exp1 exp2; do
  echo "== $v"; RMB_LIB_PATH=exp/librmb_$v.so timeout 120 python tools/ab_tma.py 10000,1000,64 2>&1 | grep "^tma"
done
