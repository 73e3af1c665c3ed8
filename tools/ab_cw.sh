for v in default cw16; do
  if [ $v = default ]; then L=""; else L="RMB_LIB_PATH=exp/librmb_$v.so"; fi
  echo "== $v"; env $L timeout 200 python tools/ab_tma.py 10000,1000,250,64,1 2>&1 | grep "^tma"
done
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_shard.py -x -q 2>&1 | tail -2
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_2110_02901_b200 as rmb, time
P,c = rmb.generate_dense(10000,16,1)
p = rmb.Problem.dense(P,c,0.99)
p.vi(1000, seed=0, eps=1e-6, max_sweeps=5)
for rep in range(3):
    s = p.vi(1000, seed=rep, eps=1e-6, max_sweeps=100000)
    print('full solve b=1000', s.stats.sweeps, round(s.stats.seconds*1e3,1), 'ms', round(s.stats.sweeps*6.4008e9/s.stats.seconds/1e9), 'GB/s')
"
