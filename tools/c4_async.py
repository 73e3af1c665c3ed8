import sys, json
sys.path.insert(0, '.')
import paper_2110_02901_b200 as rmb
N = 2048
n = N * N
rp, col, val, c = rmb.generate_grid(N)
prob = rmb.Problem.csr(n, 4, rp, col, val, c, 0.95)
prob.mpi(65536, 10, seed=0, eps=1e-6, max_outer=2)
for name, kw in (("MB-MPI b=65536", {}), ("async MB-MPI", {"asynchronous": True}), ("MB-MPI b=n", {"b": n})):
    b = kw.pop("b", 65536)
    sol = prob.mpi(b, 10, seed=0, eps=1e-6, max_outer=100_000, **kw)
    st = sol.stats
    print(json.dumps({"row": name, "status": int(sol.status), "outer": st.outer_iters, "eval_sweeps": st.sweeps,
                      "time_ms": st.seconds * 1e3, "ms_per_eval_sweep_incl_improve": st.seconds * 1e3 / st.sweeps}), flush=True)
