"""CPU oracle for the randomized mini-batch operator (arXiv 2110.02901).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
path (paper_2110_02901_b200/) never imports it, and nothing here imports the
product path.  The one shared module is gen/ (instance definition only).

Two parts:
  * oracle.c (ctypes): the method itself, step by step in the paper's order
    (partition, B_b / B_{pi,b} sweeps, MB-VI, MB-MPI) — see that file.
  * numpy extras (this file): the plain *definitions* the method converges to,
    used to pin the sweep engine: exact policy evaluation J_mu = (I - a P_mu)^-1
    g_mu (Eq. 4), brute-force J* = min over all |A|^n policies
    (Eq. 2), exact policy iteration.

Arrays: dense P is float32/float64 [n][A][n]; c is [n][A] of the same dtype;
CSR rows r = s*A + a with int64 row_ptr[n*A+1], int32 col, val like P.
V is float64 [n], policies int32 [n].
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RMB_ORACLE_SO: a prebuilt alternative oracle (tools/mutation_check.py loads
# deliberately broken builds to show that the pins catch each mutation)
_SO = os.environ.get("RMB_ORACLE_SO") or os.path.join(_HERE, "liboracle.so")
_lib = None

OK, INVALID_ARG, NOT_CONVERGED, NONFINITE, OOM = 0, 1, 3, 4, 7


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if os.environ.get("RMB_ORACLE_SO"):
        return _SO
    hdr = os.path.join(os.path.dirname(_HERE), "gen", "rmb_gen.h")
    if force or not os.path.exists(_SO) or max(os.path.getmtime(src), os.path.getmtime(hdr)) > os.path.getmtime(_SO):
        # -ffp-contract=off: no FMA contraction — every product and sum is
        # rounded exactly as written in oracle.c
        # -fopenmp: optional worker threads across the states of one batch
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
                               "-o", _SO, src, "-lm"])
    return _SO


class _Mdp(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("A", ctypes.c_int32), ("kind", ctypes.c_int32),
        ("gamma", ctypes.c_double), ("p_f32", ctypes.c_int32), ("c_f32", ctypes.c_int32),
        ("P", ctypes.c_void_p), ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p),
        ("val", ctypes.c_void_p), ("c", ctypes.c_void_p),
    ]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, i32, vp, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double
        pm = ctypes.POINTER(_Mdp)
        lib.orc_mix64.argtypes, lib.orc_mix64.restype = [u64], u64
        lib.orc_partition.argtypes = [i64, u64, i64, ctypes.c_int, vp]
        lib.orc_partition_inverse.argtypes = [i64, u64, i64, ctypes.c_int, vp]
        lib.orc_sweep.argtypes = [pm, i64, vp, vp, vp, vp, vp]
        lib.orc_sweep_chunked.argtypes = [pm, i64, vp, vp, vp, vp, vp]
        lib.orc_set_threads.argtypes, lib.orc_set_threads.restype = [ctypes.c_int], None
        lib.orc_get_threads.argtypes, lib.orc_get_threads.restype = [], ctypes.c_int
        lib.orc_improve.argtypes = [pm, vp, vp, vp, vp]
        lib.orc_vi.argtypes = [pm, i64, u64, ctypes.c_int, i64, dbl, i64, ctypes.c_int, vp, vp, vp, vp,
                               ctypes.c_int, vp]
        lib.orc_mpi.argtypes = [pm, i64, i32, u64, ctypes.c_int, i64, dbl, i64, ctypes.c_int,
                                vp, vp, vp, vp, vp, vp, ctypes.c_int, vp]
        lib.orc_select.argtypes, lib.orc_select.restype = [i64, u64, i64, vp, vp], ctypes.c_int
        lib.orc_backup_dense_row.argtypes = [i64, i32, dbl, ctypes.c_int, vp, vp, vp, i32, vp]
        lib.orc_backup_dense_row.restype = dbl
        lib.orc_backup_csr_row.argtypes = [i64, i32, dbl, ctypes.c_int, vp, vp, vp, vp, vp, i32, vp]
        lib.orc_backup_csr_row.restype = dbl
        lib.orc_bellman_residual_dense_gen.argtypes = [u64, i64, i32, ctypes.c_int, dbl, vp, i64, i64, vp]
        lib.orc_bellman_residual_dense_gen.restype = dbl
        for f in (lib.orc_partition, lib.orc_partition_inverse, lib.orc_sweep, lib.orc_sweep_chunked, lib.orc_improve,
                  lib.orc_vi, lib.orc_mpi):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


@dataclass
class MDP:
    """A finite discounted MDP (S, U, P, g, alpha) with uniform |A|."""
    n: int
    A: int
    gamma: float
    c: np.ndarray                   # [n][A]
    P: np.ndarray | None = None     # dense [n][A][n]
    row_ptr: np.ndarray | None = None
    col: np.ndarray | None = None
    val: np.ndarray | None = None

    def __post_init__(self):
        self.c = np.ascontiguousarray(self.c)
        if self.P is not None:
            self.P = np.ascontiguousarray(self.P)
            assert self.P.shape == (self.n, self.A, self.n) and self.P.dtype in (np.float32, np.float64)
        else:
            self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
            self.col = np.ascontiguousarray(self.col, dtype=np.int32)
            self.val = np.ascontiguousarray(self.val)
            assert self.row_ptr.shape == (self.n * self.A + 1,)
        assert self.c.shape == (self.n, self.A)
        pdt = (self.P if self.P is not None else self.val).dtype
        self._s = _Mdp(self.n, self.A, 0 if self.P is not None else 1, float(self.gamma),
                       int(pdt == np.float32), int(self.c.dtype == np.float32),
                       self.P.ctypes.data if self.P is not None else None,
                       self.row_ptr.ctypes.data if self.row_ptr is not None else None,
                       self.col.ctypes.data if self.col is not None else None,
                       self.val.ctypes.data if self.val is not None else None,
                       self.c.ctypes.data)

    @property
    def dense(self) -> bool:
        return self.P is not None

    def to_dense64(self) -> np.ndarray:
        """P as a float64 [n][A][n] array (exact widening / CSR scatter)."""
        if self.P is not None:
            return self.P.astype(np.float64)
        P = np.zeros((self.n * self.A, self.n))
        for r in range(self.n * self.A):
            for e in range(self.row_ptr[r], self.row_ptr[r + 1]):
                P[r, self.col[e]] += float(self.val[e])
        return P.reshape(self.n, self.A, self.n)


def set_threads(w: int) -> None:
    """Worker threads for the states of one batch / the improvement (results
    are bitwise independent of w: every per-state row sum stays sequential)."""
    _load().orc_set_threads(int(w))


def get_threads() -> int:
    return int(_load().orc_get_threads())


# ---------------------------------------------------------------- partition
def mix64(z: int) -> int:
    return int(_load().orc_mix64(z & (2**64 - 1)))


def partition(n: int, seed: int, k: int, identity: bool = False) -> np.ndarray:
    """perm[p] = pi_k(p), the state at position p of sweep k."""
    out = np.empty(n, dtype=np.uint32)
    rc = _load().orc_partition(n, seed, k, int(identity), _p(out))
    if rc:
        raise ValueError("partition: invalid argument")
    return out


def partition_inverse(n: int, seed: int, k: int, identity: bool = False) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    rc = _load().orc_partition_inverse(n, seed, k, int(identity), _p(out))
    if rc:
        raise ValueError("partition_inverse: invalid argument")
    return out


def select(n: int, seed: int, k: int, weights: np.ndarray | None = None) -> np.ndarray:
    """The n states drawn WITH replacement for operator application k (DESIGN
    R28-R29): uniform, or P(s) = w_s / sum(w) for
    integer weights w_s >= 1."""
    out = np.empty(n, dtype=np.uint32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.uint32)
    if w is not None and w.shape != (n,):
        raise ValueError("select: weights must have n entries")
    rc = _load().orc_select(n, seed, k, _p(w), _p(out))
    if rc:
        raise ValueError("select: invalid argument (n out of range or a zero weight)")
    return out


def _sel_args(select, weights, n):
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.uint32)
        assert w.shape == (n,)
        return 1, w
    return int(bool(select)), None


# ------------------------------------------------------------ the operator
def sweep(m: MDP, V: np.ndarray, b: int, perm: np.ndarray, pi: np.ndarray | None = None):
    """One application of B_b (pi None) or B_{pi,b}: returns (V', argmin, r)."""
    V = np.array(V, dtype=np.float64, copy=True)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    arg = np.zeros(m.n, dtype=np.int32)
    pi_c = np.ascontiguousarray(pi, dtype=np.int32) if pi is not None else None
    r = ctypes.c_double()
    rc = _load().orc_sweep(ctypes.byref(m._s), b, _p(perm), _p(pi_c), _p(V), _p(arg), ctypes.byref(r))
    if rc not in (OK, NONFINITE):
        raise ValueError(f"sweep: status {rc}")
    return V, arg, r.value


def sweep_chunked(m: MDP, V: np.ndarray, c: int, perm: np.ndarray, pi: np.ndarray | None = None):
    """VI*'s operator: T (or T_pi) in chunks of c states against the
    old values; returns (V', argmin, r)."""
    V = np.array(V, dtype=np.float64, copy=True)
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    arg = np.zeros(m.n, dtype=np.int32)
    pi_c = np.ascontiguousarray(pi, dtype=np.int32) if pi is not None else None
    r = ctypes.c_double()
    rc = _load().orc_sweep_chunked(ctypes.byref(m._s), c, _p(perm), _p(pi_c), _p(V), _p(arg), ctypes.byref(r))
    if rc not in (OK, NONFINITE):
        raise ValueError(f"sweep_chunked: status {rc}")
    return V, arg, r.value


def improve(m: MDP, V: np.ndarray, pi: np.ndarray):
    """Policy improvement: returns (pi', ||TV-V||_inf, changed)."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    pi2 = np.array(pi, dtype=np.int32, copy=True)
    r, ch = ctypes.c_double(), ctypes.c_int64()
    rc = _load().orc_improve(ctypes.byref(m._s), _p(V), _p(pi2), ctypes.byref(r), ctypes.byref(ch))
    if rc not in (OK, NONFINITE):
        raise ValueError(f"improve: status {rc}")
    return pi2, r.value, ch.value


@dataclass
class Result:
    status: int
    V: np.ndarray
    pi: np.ndarray
    trace: np.ndarray
    sweeps: int
    outer: int = 0
    changed: np.ndarray | None = None


def vi(m: MDP, b: int, seed: int = 0, eps: float = 1e-6, max_sweeps: int = 100000,
       V0: np.ndarray | None = None, identity: bool = False, first_sweep: int = 1,
       chunked: bool = False, replace: bool = False, weights: np.ndarray | None = None) -> Result:
    """MB-VI to ||V_k - V_{k-1}||_inf <= eps; chunked=True: VI* (P:L577),
    T in chunks of b states against the old values; replace=True / weights:
    every sweep draws n states with replacement (uniform / P(s) ~ w_s, R28-R29)."""
    V = np.zeros(m.n) if V0 is None else np.array(V0, dtype=np.float64, copy=True)
    pi = np.zeros(m.n, dtype=np.int32)
    tr = np.zeros(max_sweeps)
    sw = ctypes.c_int64()
    sel, w = _sel_args(replace, weights, m.n)
    st = _load().orc_vi(ctypes.byref(m._s), b, seed, int(identity), first_sweep, eps, max_sweeps,
                        int(chunked), _p(V), _p(pi), _p(tr), ctypes.byref(sw), sel, _p(w))
    if st == INVALID_ARG:
        raise ValueError("vi: invalid argument")
    return Result(st, V, pi, tr[: sw.value], sw.value)


def mpi(m: MDP, b: int, msweeps: int, seed: int = 0, eps: float = 1e-6, max_outer: int = 10000,
        V0: np.ndarray | None = None, pi0: np.ndarray | None = None, identity: bool = False,
        first_sweep: int = 1, replace: bool = False, weights: np.ndarray | None = None) -> Result:
    """MB-MPI: Algorithm 1 with B_{pi,b} evaluation and warm start
    (replace / weights: evaluation sweeps draw with replacement, R28-R29)."""
    V = np.zeros(m.n) if V0 is None else np.array(V0, dtype=np.float64, copy=True)
    pi = np.zeros(m.n, dtype=np.int32) if pi0 is None else np.array(pi0, dtype=np.int32, copy=True)
    tr = np.zeros(max_outer * (msweeps + 1))
    chg = np.zeros(max_outer, dtype=np.int64)
    sw, ou = ctypes.c_int64(), ctypes.c_int64()
    sel, w = _sel_args(replace, weights, m.n)
    st = _load().orc_mpi(ctypes.byref(m._s), b, msweeps, seed, int(identity), first_sweep, eps, max_outer,
                         int(pi0 is not None), _p(V), _p(pi), _p(tr), _p(chg), ctypes.byref(sw),
                         ctypes.byref(ou), sel, _p(w))
    if st == INVALID_ARG:
        raise ValueError("mpi: invalid argument")
    o = ou.value
    return Result(st, V, pi, tr[: o * (msweeps + 1)], sw.value, o, chg[:o])


def backup_dense_row(P_rows: np.ndarray, c_row: np.ndarray, gamma: float, Vint: np.ndarray,
                     pi_a: int = -1):
    """(Q_min or Q_pi, argmin) of one state from its [A][n] rows and an explicit interim V."""
    P_rows = np.ascontiguousarray(P_rows)
    c_row = np.ascontiguousarray(c_row, dtype=P_rows.dtype)
    A, n = P_rows.shape
    Vint = np.ascontiguousarray(Vint, dtype=np.float64)
    arg = ctypes.c_int32()
    q = _load().orc_backup_dense_row(n, A, gamma, int(P_rows.dtype == np.float32), _p(P_rows), _p(c_row),
                                     _p(Vint), pi_a, ctypes.byref(arg))
    return q, arg.value


def backup_csr_row(n: int, row_ptr: np.ndarray, col: np.ndarray, val: np.ndarray, c_row: np.ndarray,
                   gamma: float, Vint: np.ndarray, pi_a: int = -1):
    """(Q_min or Q_pi, argmin) of one state from its A CSR rows (row_ptr: A+1 offsets)."""
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val)
    c_row = np.ascontiguousarray(c_row, dtype=val.dtype)
    Vint = np.ascontiguousarray(Vint, dtype=np.float64)
    arg = ctypes.c_int32()
    q = _load().orc_backup_csr_row(n, len(row_ptr) - 1, gamma, int(val.dtype == np.float32), _p(row_ptr), _p(col),
                                   _p(val), _p(c_row), _p(Vint), pi_a, ctypes.byref(arg))
    return q, arg.value


def bellman_residual_dense_gen(seed: int, n: int, A: int, gamma: float, V: np.ndarray, rows=None,
                               f32: bool = True):
    """||T V - V||_inf over rows (s0, s1) of the dense random instance (seed, n, A),
    its rows regenerated on the host (certificate ||V - V*|| <= r / (1 - gamma),
    Prop. 3).  Returns (r, argmin over the rows)."""
    s0, s1 = rows if rows is not None else (0, n)
    V = np.ascontiguousarray(V, dtype=np.float64)
    arg = np.zeros(s1 - s0, dtype=np.int32)
    r = _load().orc_bellman_residual_dense_gen(seed, n, A, int(f32), gamma, _p(V), s0, s1, _p(arg))
    return r, arg


# ------------------------------------------------- plain definitions (numpy)
def policy_value(m: MDP, mu: np.ndarray) -> np.ndarray:
    """J_mu solving J = g_mu + alpha P_mu J (Eq. 4), dense fp64 solve."""
    P = m.to_dense64()
    idx = np.arange(m.n)
    Pmu = P[idx, mu, :]
    gmu = m.c.astype(np.float64)[idx, mu]
    return np.linalg.solve(np.eye(m.n) - m.gamma * Pmu, gmu)


def brute_force(m: MDP):
    """J* = min over all stationary policies of J_mu (Eq. 2), mu* = the
    lexicographically first minimiser per state.  |A|^n policies: tiny MDPs only."""
    assert m.A ** m.n <= 20000, "brute force is for tiny MDPs"
    best = None
    for mu in itertools.product(range(m.A), repeat=m.n):
        J = policy_value(m, np.array(mu))
        best = J if best is None else np.minimum(best, J)
    return best


def policy_iteration(m: MDP, max_iter: int = 1000):
    """Exact PI: alternate J_mu (linear solve) and greedy improvement."""
    P = m.to_dense64()
    c = m.c.astype(np.float64)
    mu = np.zeros(m.n, dtype=np.int64)
    for _ in range(max_iter):
        J = policy_value(m, mu)
        Q = c + m.gamma * np.einsum("saj,j->sa", P, J)
        new = mu.copy()
        for s in range(m.n):   # keep mu(s) unless strictly improvable (termination)
            a = int(np.argmin(Q[s]))
            if Q[s, a] < Q[s, mu[s]] - 1e-13 * max(1.0, abs(Q[s, a])):
                new[s] = a
        if np.array_equal(new, mu):
            return J, mu.astype(np.int32)
        mu = new
    raise RuntimeError("policy iteration did not terminate")
