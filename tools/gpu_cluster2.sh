RMB_CLUSTER_DEBUG=1 timeout 300 python tools/ab_tma.py 1 2>&1 | grep -E "cluster" | tail -4
