"""RMB_TRACE_ERROR_VS_REF (the paper's plotted metric
||V_k - V*||_inf): the device-recorded error after every
operator application, on every solver path, against the oracle.

Per sweep the error is a max of |V_k(s) - V*(s)| (exact in fp64), so it
differs from the oracle's only through V_k itself (1e-11 relative per
application, R16); the last entry is bitwise the host's max over the
returned V.
"""
import numpy as np
import pytest
import torch

import gen
import oracle
import paper_2110_02901_b200 as rmb

pytestmark = pytest.mark.gpu


def tdev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def dense(n, A, seed, flags=0, gamma=0.9):
    P, c = gen.dense(n, A, seed, dtype=np.float32)
    return oracle.MDP(n, A, gamma, c, P=P), rmb.Problem.dense(tdev(P), tdev(c), gamma, flags=flags)


def sparse():
    rp, col, val, c = gen.grid(16)
    m = oracle.MDP(256, 4, 0.95, c, row_ptr=rp, col=col, val=val)
    return m, rmb.Problem.csr(256, 4, tdev(rp), tdev(col), tdev(val), tdev(c), 0.95)


CASES = {"dense_grid": lambda: dense(300, 8, 1, rmb.DENSE_NO_CLUSTER), "dense_cluster": lambda: dense(300, 8, 1),
         "dense_vglobal": lambda: dense(300, 8, 1, rmb.DENSE_VGLOBAL | rmb.DENSE_NO_CLUSTER),
         "dense_warp": lambda: dense(300, 8, 1, rmb.DENSE_NO_TMA), "sparse": sparse}


def oracle_errors(m, b, seed, sweeps, Vref):
    V, out = np.zeros(m.n), []
    for k in range(1, sweeps + 1):
        V = oracle.sweep(m, V, b, oracle.partition(m.n, seed, k))[0]
        out.append(np.abs(V - Vref).max())
    return np.array(out)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("b", [1, 3, 37])   # b = 1 on the cluster path: the look-ahead kernel
def test_error_trace_matches_oracle(name, b):
    m, prob = CASES[name]()
    Vref = oracle.vi(m, m.n, eps=1e-13, max_sweeps=100000, identity=True).V
    prob.set_reference(tdev(Vref))
    sol = prob.vi(b, seed=4, eps=1e-8, max_sweeps=3000, trace_error=True)
    assert sol.status == rmb.OK
    err = sol.error
    assert len(err) == sol.stats.sweeps
    ref = oracle_errors(m, b, 4, sol.stats.sweeps, Vref)
    scale = max(1.0, np.abs(Vref).max())
    assert np.abs(err - ref).max() <= 1e-10 * scale
    assert err[-1] == np.abs(sol.V.cpu().numpy() - Vref).max()   # the same fp64 max, bitwise


@pytest.mark.parametrize("mode", ["async", "replace", "mpi", "policy"])
@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_error_trace_other_solves(mode, kind):
    m, prob = dense(300, 8, 1) if kind == "dense" else sparse()
    Vref = oracle.vi(m, m.n, eps=1e-13, max_sweeps=100000, identity=True).V
    prob.set_reference(Vref)   # host reference
    if mode == "policy":
        pi = tdev(np.zeros(m.n, np.int32))
        J = oracle.policy_value(m, np.zeros(m.n, np.int32))
        prob.set_reference(tdev(J))
        flags = rmb.TRACE_ERROR_VS_REF | rmb.V0_ZERO
        V = torch.zeros(m.n, dtype=torch.float64, device="cuda")
        st = rmb.Stats()
        s = rmb.lib().rmb_policy_value(prob._h, rmb._ptr(pi), 17, 0, 1e-10, 5000, flags, rmb._ptr(V), None,
                                       rmb.ctypes.byref(st))
        assert s == rmb.OK
        err = prob.error_trace()
        assert len(err) == st.sweeps and err[-1] == np.abs(V.cpu().numpy() - J).max()
        return
    if mode == "mpi":
        sol = prob.mpi(37, 4, seed=2, eps=1e-9, trace_error=True)
    else:
        sol = prob.vi(37, seed=2, eps=1e-9, max_sweeps=5000, trace_error=True,
                      **({"asynchronous": True} if mode == "async" else {"select": "replace"}))
    assert sol.status == rmb.OK
    err = sol.error
    assert len(err) == sol.stats.sweeps
    assert err[-1] == np.abs(sol.V.cpu().numpy() - Vref).max()
    assert err[-1] < 1e-6 and err[0] > err[-1]
    if mode == "async":   # from V0 = 0 with costs >= 0 the iterates rise monotonically to V*
        assert (np.diff(err) <= 1e-12).all()


def test_error_trace_needs_a_reference():
    m, prob = dense(64, 4, 2)
    with pytest.raises(rmb.RmbError):
        prob.vi(8, trace_error=True)
    prob.set_reference(np.zeros(64))
    prob.vi(8, eps=1e-6, trace_error=True)
    prob.vi(8, eps=1e-6)
    assert len(prob.error_trace()) == 0   # the last solve did not trace
