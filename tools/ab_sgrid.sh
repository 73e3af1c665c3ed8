for g in 1 2 8 148; do
  echo "== grid $g"; RMB_SPARSE_GRID=$g timeout 300 python tools/env_bench.py 2>&1 | tr -d '\n' | sed 's/}/}\n/g' | grep -o '"b": [0-9]*, *"sweeps": [0-9]*, *"time_to_eps_ms": [0-9.]*' | tr '\n' ' '; echo
done
