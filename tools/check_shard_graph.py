import sys; sys.path.insert(0,'.')
import numpy as np, torch, gen, paper_2110_02901_b200 as rmb
N=16; n=N*N; rp,col,val,c=gen.grid(N,dtype=np.float32)
def t(x): return torch.from_numpy(np.ascontiguousarray(x)).cuda()
hs=[]
for g in range(2):
    r0,r1=rmb.shard_range(n,2,g); e0,e1=rp[r0*4],rp[r1*4]
    hs.append(rmb.Problem.csr(n,4,t(rp[r0*4:r1*4+1]-e0),t(col[e0:e1]),t(val[e0:e1]),t(c[r0:r1]),0.95,row_range=(r0,r1)))
print("sparse group", rmb.vi_group(hs,23,seed=1,eps=1e-9,max_sweeps=20).stats.sweeps, flush=True)
P,c=gen.dense(200,4,1,dtype=np.float32)
hs=[rmb.Problem.dense(t(P[a:b]),t(c[a:b]),0.95,n=200,row_range=(a,b)) for a,b in [rmb.shard_range(200,2,g) for g in range(2)]]
print("dense group", rmb.vi_group(hs,23,seed=1,eps=1e-9,max_sweeps=20).stats.sweeps, flush=True)
