for cfg in "" "RMB_TMA_G=4" "RMB_TMA_HINT=0" "RMB_TMA_NST=3" "RMB_TMA_NST=2" "RMB_TMA_G=8 RMB_TMA_HINT=0"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/ab_tma.py 10000,1000 2>&1 | grep "^tma"
done
timeout 120 python tools/prof_dense.py 10000 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_solver -c 1 -o gpurun_out/dense_tma_bn python tools/prof_dense.py 10000 3 > gpurun_out/ncu_tma.log 2>&1; echo ncu rc=$?
