timeout 200 python tools/ab_tma.py 10000,1000,250,64,1 2>&1 | grep -v "^warp"
for cfg in "RMB_TMA_IPSM=4" "RMB_TMA_IPSM=8" "RMB_TMA_REDUNDANT_MAX=8192" "RMB_TMA_STATIC=4" "RMB_TMA_IPSM=1"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/ab_tma.py 1000,250,64,1 2>&1 | grep "^tma"
done
