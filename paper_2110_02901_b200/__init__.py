"""paper_2110_02901_b200 — B200-native randomized mini-batch dynamic programming.

Thin ctypes binding over librmb.so (include/rmb.h).  Argument marshalling
only: every step of the method (partition, batched backups, residuals, stop
test, policy improvement) runs in the library's sm_100a CUDA kernels.  PyTorch
supplies device memory and streams.  There is no CPU fallback: if librmb.so is
missing or fails to load, every call raises.

    import paper_2110_02901_b200 as rmb
    P, c = rmb.generate_dense(n=10_000, A=16, seed=1)          # on cuda
    prob = rmb.Problem.dense(P, c, gamma=0.99)
    out = prob.vi(b=1000, seed=0, eps=1e-6)                      # MB-VI
    out = prob.mpi(b=1000, m=10, seed=0, eps=1e-6)               # MB-MPI (Alg. 1)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMB_LIB_PATH") or os.path.join(_HERE, "librmb.so")  # override: experiments only

# status codes (include/rmb.h)
OK, INVALID_ARG, INVALID_MDP, NOT_CONVERGED, NONFINITE, CUDA_ERR, NCCL_ERR, OOM, UNSUPPORTED = range(9)
F32, F64 = 0, 1
ORDER_IDENTITY, V0_ZERO, PI_GIVEN, VALIDATE, DENSE_NO_TMA, DENSE_VGLOBAL = 0x1, 0x2, 0x4, 0x8, 0x10, 0x20
CHUNKED_T = 0x40
SPARSE_FULL_GRID, SHARD_NO_GRAPH, FUSED, DENSE_NO_CLUSTER = 0x80, 0x400, 0x800, 0x1000
SELECT_REPLACE, SELECT_WEIGHTED, ASYNC = 0x2000, 0x4000, 0x8000
TRACE_ERROR_VS_REF = 0x10000

_lib = None


class RmbError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_status_name(status)}: {msg}")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [("n_states", ctypes.c_int64), ("n_actions", ctypes.c_int32), ("gamma", ctypes.c_double),
                ("p_dtype", ctypes.c_int), ("v_dtype", ctypes.c_int), ("row_begin", ctypes.c_int64),
                ("row_end", ctypes.c_int64), ("nccl_comm", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("sweeps", ctypes.c_int64), ("batches", ctypes.c_int64), ("outer_iters", ctypes.c_int64),
                ("final_residual", ctypes.c_double), ("seconds", ctypes.c_double),
                ("converged", ctypes.c_int32), ("status", ctypes.c_int32)]


_SIGS = {
    "rmb_create_dense": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                          ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "rmb_create_csr": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "rmb_vi": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int64,
                ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)],
               ctypes.c_int),
    "rmb_mpi": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double,
                 ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                 ctypes.c_void_p, ctypes.POINTER(Stats)], ctypes.c_int),
    "rmb_apply": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                   ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "rmb_policy_value": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                          ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)],
                         ctypes.c_int),
    "rmb_improve": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                     ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "rmb_partition": ([ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p],
                      ctypes.c_int),
    "rmb_partition_device": ([ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32,
                              ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_generate_dense": ([ctypes.c_int32, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                            ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
                           ctypes.c_int),
    "rmb_generate_sparse": ([ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                             ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_generate_grid": ([ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_last_launch_count": ([ctypes.c_void_p], ctypes.c_int64),
    "rmb_last_graph_launches": ([ctypes.c_void_p], ctypes.c_int64),
    "rmb_shard_range": ([ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                         ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "rmb_nccl_unique_id": ([ctypes.c_void_p], ctypes.c_int),
    "rmb_nccl_comm_init": ([ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)],
                           ctypes.c_int),
    "rmb_nccl_comm_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "rmb_vi_group": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                      ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.POINTER(Stats)], ctypes.c_int),
    "rmb_mpi_group": ([ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                       ctypes.c_uint64, ctypes.c_double, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Stats)], ctypes.c_int),
    "rmb_last_phase_times": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_set_selection_weights": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_set_reference": ([ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_error_trace": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
                        ctypes.c_int),
    "rmb_select": ([ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "rmb_select_device": ([ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p],
                          ctypes.c_int),
    "rmb_destroy": ([ctypes.c_void_p], ctypes.c_int),
    "rmb_status_string": ([ctypes.c_int], ctypes.c_char_p),
    "rmb_last_error": ([], ctypes.c_char_p),
    "rmb_version": ([], ctypes.c_char_p),
}


def lib():
    """Load librmb.so (building it first if the sources are newer). Raises if unavailable."""
    global _lib
    if _lib is None:
        from . import _build
        if LIB_PATH == _build.SO and _build.needs_build():
            _build.build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"librmb.so not found at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


def _status_name(s):
    try:
        return lib().rmb_status_string(s).decode()
    except Exception:
        return str(s)


def _check(status, ok=(OK,)):
    if status not in ok:
        raise RmbError(status, lib().rmb_last_error().decode())
    return status


# ------------------------------------------------------------------ buffers
def _ptr(x):
    """Raw address of a torch tensor / numpy array (host or device), or None."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return ctypes.c_void_p(x.ctypes.data)
    assert x.is_contiguous()
    return ctypes.c_void_p(x.data_ptr())


def _vec(x, n, kind, what):
    """Check a V (kind "f64") or pi (kind "i32") buffer: dtype and length n.
    The library reads / writes exactly n elements of that type."""
    if x is None:
        return x
    import torch
    want = {"f64": (np.float64, torch.float64), "i32": (np.int32, torch.int32)}[kind]
    if x.dtype not in want:
        raise TypeError(f"{what} must be {'float64' if kind == 'f64' else 'int32'}, got {x.dtype}")
    numel = x.size if isinstance(x, np.ndarray) else x.numel()
    if numel != n:
        raise ValueError(f"{what} must have n = {n} elements, got {numel}")
    return x


def _dtype_code(x):
    import torch
    dt = x.dtype
    if dt in (np.float32, torch.float32):
        return F32
    if dt in (np.float64, torch.float64):
        return F64
    raise TypeError(f"P/c must be float32 or float64, got {dt}")


def _stream_ptr(stream):
    import torch
    if stream is None:
        if not torch.cuda.is_available():
            return None
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


@dataclass
class Solution:
    V: object
    pi: object
    trace: np.ndarray
    status: int
    stats: Stats
    changed: np.ndarray | None = None
    error: np.ndarray | None = None   # ||V_i - V*||_inf per application (trace_error=True)

    @property
    def converged(self):
        return self.status == OK


class Problem:
    """A handle over an MDP (S, U, P, g, alpha) living on the GPU."""

    def __init__(self, handle, n, A, gamma, keep):
        self._h = handle
        self.n, self.A, self.gamma = n, A, gamma
        self._keep = keep  # borrowed buffers must outlive the handle

    # ------------------------------------------------------------ creation
    @classmethod
    def dense(cls, P, c, gamma, stream=None, validate=False, n=None, row_range=None, nccl_comm=None, tma=True,
              vglobal=False, flags=0):
        """P: [n][A][n], c: [n][A] (float32/float64, torch cuda/cpu or numpy).
        Shard handle (multi-GPU): P = the owned rows [r1-r0][A][n], c = [r1-r0][A],
        n = the global state count, row_range = (r0, r1) from shard_range(),
        nccl_comm = comm_init(...) (or None for a logical group on one GPU).
        tma=False: RMB_DENSE_NO_TMA (register-streaming warp path instead of the TMA ring).
        vglobal=True: RMB_DENSE_VGLOBAL (V and pi in global memory; automatic for large n)."""
        rows, A, ncol = P.shape
        n = ncol if n is None else n
        r0, r1 = row_range if row_range is not None else (0, n)
        assert ncol == n and rows == r1 - r0 and tuple(c.shape) == (rows, A) and c.dtype == P.dtype
        d = _Desc(n, A, float(gamma), _dtype_code(P), F64, r0, r1, nccl_comm, _stream_ptr(stream))
        h = ctypes.c_void_p()
        flags |= (VALIDATE if validate else 0) | (0 if tma else DENSE_NO_TMA) | (DENSE_VGLOBAL if vglobal else 0)
        _check(lib().rmb_create_dense(ctypes.byref(d), _ptr(P), _ptr(c), flags, ctypes.byref(h)))
        return cls(h, n, A, float(gamma), (P, c))

    @classmethod
    def csr(cls, n, A, row_ptr, col, val, c, gamma, stream=None, validate=False, row_range=None, nccl_comm=None,
            flags=0):
        """CSR over rows r = s*A + a: row_ptr int64 [n*A+1], col int32, val float.
        Shard handle (multi-GPU): row_range = (r0, r1) from shard_range(), row_ptr
        [(r1-r0)*A+1] from 0 over the owned rows, col GLOBAL successor ids, c [r1-r0][A];
        nccl_comm as for dense().  flags: extra create flags (SPARSE_*, SHARD_NO_GRAPH)."""
        r0, r1 = row_range if row_range is not None else (0, n)
        d = _Desc(n, A, float(gamma), _dtype_code(val), F64, r0, r1, nccl_comm, _stream_ptr(stream))
        h = ctypes.c_void_p()
        _check(lib().rmb_create_csr(ctypes.byref(d), _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(c),
                                    (VALIDATE if validate else 0) | flags, ctypes.byref(h)))
        return cls(h, n, A, float(gamma), (row_ptr, col, val, c))

    def close(self):
        if self._h:
            lib().rmb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -------------------------------------------------------------- solves
    def _vp(self, V, pi, device):
        import torch
        if V is None:
            V = torch.zeros(self.n, dtype=torch.float64, device=device)
        if pi is None:
            pi = torch.zeros(self.n, dtype=torch.int32, device=device)
        return _vec(V, self.n, "f64", "V"), _vec(pi, self.n, "i32", "pi")

    def vi(self, b, seed=0, eps=1e-6, max_sweeps=100_000, V=None, pi=None, identity=False, v0_zero=False,
           device="cuda", chunked=False, fused=False, select=None, asynchronous=False, trace_error=False):
        """MB-VI: V, pi updated in place (torch cuda/cpu or numpy).
        chunked=True: VI* -- every sweep is T computed in chunks of b
        states against the sweep-start values (RMB_CHUNKED_T).
        select="replace" / "weighted": every sweep draws n states with
        replacement, uniformly / by the weights of set_selection_weights (R28-R30).
        asynchronous=True: RMB_ASYNC (R31) -- no batch barrier, b unused.
        trace_error=True: record ||V_k - V*||_inf per sweep (set_reference first)."""
        V, pi = self._vp(V, pi, device)
        tr = np.zeros(max_sweeps)
        st = Stats()
        flags = ((ORDER_IDENTITY if identity else 0) | (V0_ZERO if v0_zero else 0) | (CHUNKED_T if chunked else 0)
                 | (FUSED if fused else 0) | _select_flag(select) | (ASYNC if asynchronous else 0)
                 | (TRACE_ERROR_VS_REF if trace_error else 0))
        s = lib().rmb_vi(self._h, b, seed, eps, max_sweeps, flags, _ptr(V), _ptr(pi), _ptr(tr), ctypes.byref(st))
        _check(s, (OK, NOT_CONVERGED, NONFINITE))
        return Solution(V, pi, tr[: st.sweeps], s, st, error=self.error_trace() if trace_error else None)

    def mpi(self, b, m, seed=0, eps=1e-6, max_outer=10_000, V=None, pi=None, pi_given=False, identity=False,
            v0_zero=False, device="cuda", fused=False, select=None, asynchronous=False, trace_error=False):
        """MB-MPI: Algorithm 1 with B_{pi,b} evaluation, warm start
        (select: evaluation sweeps draw with replacement, as vi())."""
        V, pi = self._vp(V, pi, device)
        tr = np.zeros(max_outer * (m + 1))
        ch = np.zeros(max_outer, dtype=np.int64)
        st = Stats()
        flags = ((ORDER_IDENTITY if identity else 0) | (V0_ZERO if v0_zero else 0) | (PI_GIVEN if pi_given else 0)
                 | (FUSED if fused else 0) | _select_flag(select) | (ASYNC if asynchronous else 0)
                 | (TRACE_ERROR_VS_REF if trace_error else 0))
        s = lib().rmb_mpi(self._h, b, m, seed, eps, max_outer, flags, _ptr(V), _ptr(pi), _ptr(tr), _ptr(ch),
                          ctypes.byref(st))
        _check(s, (OK, NOT_CONVERGED, NONFINITE))
        o = st.outer_iters
        return Solution(V, pi, tr[: o * (m + 1)], s, st, ch[:o], error=self.error_trace() if trace_error else None)

    def apply(self, b, seed, sweep, V_in, V_out=None, pi=None, argmin=None, identity=False, chunked=False,
              select=None, asynchronous=False):
        """One application of B_b (pi None) or B_{pi,b}: returns (V_out, argmin, residual)."""
        import torch
        _vec(V_in, self.n, "f64", "V_in")
        _vec(pi, self.n, "i32", "pi")
        if V_out is None:
            V_out = torch.empty_like(V_in) if not isinstance(V_in, np.ndarray) else np.empty_like(V_in)
        _vec(V_out, self.n, "f64", "V_out")
        if argmin is None:
            argmin = (torch.empty(self.n, dtype=torch.int32, device=V_out.device)
                      if not isinstance(V_out, np.ndarray) else np.empty(self.n, np.int32))
        _vec(argmin, self.n, "i32", "argmin")
        r = ctypes.c_double()
        flags = ((ORDER_IDENTITY if identity else 0) | (CHUNKED_T if chunked else 0) | _select_flag(select)
                 | (ASYNC if asynchronous else 0))
        s = lib().rmb_apply(self._h, b, seed, sweep, flags, _ptr(pi), _ptr(V_in),
                            _ptr(V_out), _ptr(argmin), ctypes.byref(r))
        _check(s, (OK, NONFINITE))
        return V_out, argmin, r.value

    def policy_value(self, pi, b=None, seed=0, eps=1e-10, max_sweeps=1_000_000, V=None, v0_zero=True,
                     identity=False, device="cuda", asynchronous=False):
        """J_pi by B_{pi,b} iteration to ||V_k - V_{k-1}|| <= eps (Eq. 4 / Lemma 4)."""
        import torch
        V = torch.zeros(self.n, dtype=torch.float64, device=device) if V is None else V
        _vec(V, self.n, "f64", "V")
        _vec(pi, self.n, "i32", "pi")
        tr = np.zeros(min(max_sweeps, 1 << 20))
        st = Stats()
        flags = (ORDER_IDENTITY if identity else 0) | (V0_ZERO if v0_zero else 0) | (ASYNC if asynchronous else 0)
        s = lib().rmb_policy_value(self._h, _ptr(pi), self.n if b is None else b, seed, eps, max_sweeps, flags,
                                   _ptr(V), _ptr(tr) if max_sweeps <= len(tr) else None, ctypes.byref(st))
        _check(s, (OK, NOT_CONVERGED, NONFINITE))
        return Solution(V, pi, tr[: min(st.sweeps, len(tr))], s, st)

    def improve(self, V, pi):
        """Policy improvement (Alg. 1): pi in place; returns (pi, ||TV-V||, changed)."""
        _vec(V, self.n, "f64", "V")
        _vec(pi, self.n, "i32", "pi")
        r, ch = ctypes.c_double(), ctypes.c_int64()
        s = lib().rmb_improve(self._h, _ptr(V), _ptr(pi), ctypes.byref(r), ctypes.byref(ch))
        _check(s, (OK, NONFINITE))
        return pi, r.value, ch.value

    def set_reference(self, Vref):
        """V* for trace_error (float64 [n], host or device; None clears)."""
        if Vref is not None:
            _vec(Vref, self.n, "f64", "Vref")
        _check(lib().rmb_set_reference(self._h, _ptr(Vref)))

    def error_trace(self):
        """||V_i - V*||_inf per application of the last traced solve (numpy)."""
        cnt = ctypes.c_int64()
        _check(lib().rmb_error_trace(self._h, None, 0, ctypes.byref(cnt)))
        out = np.zeros(cnt.value)
        if cnt.value:
            _check(lib().rmb_error_trace(self._h, _ptr(out), cnt.value, None))
        return out

    def set_selection_weights(self, w):
        """Integer weights w_s >= 1 ([n] uint32, host or device; None clears) for
        select="weighted": state s is drawn with probability w_s / sum(w) (R29)."""
        if w is not None:
            import torch
            if w.dtype not in (np.uint32, torch.int32, np.int32):
                raise TypeError(f"weights must be uint32 (or int32 >= 1), got {w.dtype}")
            numel = w.size if isinstance(w, np.ndarray) else w.numel()
            if numel != self.n:
                raise ValueError(f"weights must have n = {self.n} entries, got {numel}")
        _check(lib().rmb_set_selection_weights(self._h, _ptr(w)))

    def select_device(self, seed, sweep, weighted=False):
        """The draws of application `sweep` from the solvers' device kernel (cuda int32 tensor)."""
        import torch
        out = torch.empty(self.n, dtype=torch.int32, device="cuda")
        _check(lib().rmb_select_device(self._h, seed, sweep, SELECT_WEIGHTED if weighted else SELECT_REPLACE,
                                       _ptr(out)))
        return out

    def last_launch_count(self):
        return int(lib().rmb_last_launch_count(self._h))

    def last_graph_launches(self):
        return int(lib().rmb_last_graph_launches(self._h))

    def last_phase_times(self):
        """(compute_ns, barrier_ns, combine_ns, n_barriers) of the last solve, CTA 0's view."""
        out = np.zeros(4, dtype=np.int64)
        _check(lib().rmb_last_phase_times(self._h, _ptr(out)))
        return tuple(int(x) for x in out)


# ------------------------------------------------------------ multi-GPU
def shard_range(n, G, g):
    """Owned rows [begin, end) of rank g of G (contiguous blocks of ceil(n/G))."""
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().rmb_shard_range(n, G, g, ctypes.byref(b), ctypes.byref(e)))
    return b.value, e.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().rmb_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_init(nranks, rank, uid: bytes):
    """ncclComm_t (as an int) for desc.nccl_comm; uid from rank 0's nccl_unique_id()."""
    comm = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(lib().rmb_nccl_comm_init(nranks, rank, buf, ctypes.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm):
    _check(lib().rmb_nccl_comm_destroy(comm))


def _handles(problems):
    arr = (ctypes.c_void_p * len(problems))(*[p._h.value if isinstance(p._h, ctypes.c_void_p) else p._h
                                              for p in problems])
    return arr


def vi_group(problems, b, seed=0, eps=1e-6, max_sweeps=100_000, V=None, pi=None, identity=False, v0_zero=False,
             device="cuda", fused=False):
    """MB-VI over G logical shard handles on one GPU (device-copy exchange)."""
    import torch
    n = problems[0].n
    V = torch.zeros(n, dtype=torch.float64, device=device) if V is None else V
    pi = torch.zeros(n, dtype=torch.int32, device=device) if pi is None else pi
    _vec(V, n, "f64", "V")
    _vec(pi, n, "i32", "pi")
    tr = np.zeros(max_sweeps)
    st = Stats()
    flags = (ORDER_IDENTITY if identity else 0) | (V0_ZERO if v0_zero else 0) | (FUSED if fused else 0)
    s = lib().rmb_vi_group(_handles(problems), len(problems), b, seed, eps, max_sweeps, flags, _ptr(V), _ptr(pi),
                           _ptr(tr), ctypes.byref(st))
    _check(s, (OK, NOT_CONVERGED, NONFINITE))
    return Solution(V, pi, tr[: st.sweeps], s, st)


def mpi_group(problems, b, m, seed=0, eps=1e-6, max_outer=10_000, V=None, pi=None, pi_given=False, identity=False,
              v0_zero=False, device="cuda", fused=False):
    """MB-MPI over G logical shard handles on one GPU."""
    import torch
    n = problems[0].n
    V = torch.zeros(n, dtype=torch.float64, device=device) if V is None else V
    pi = torch.zeros(n, dtype=torch.int32, device=device) if pi is None else pi
    _vec(V, n, "f64", "V")
    _vec(pi, n, "i32", "pi")
    tr = np.zeros(max_outer * (m + 1))
    ch = np.zeros(max_outer, dtype=np.int64)
    st = Stats()
    flags = ((ORDER_IDENTITY if identity else 0) | (V0_ZERO if v0_zero else 0) | (PI_GIVEN if pi_given else 0)
             | (FUSED if fused else 0))
    s = lib().rmb_mpi_group(_handles(problems), len(problems), b, m, seed, eps, max_outer, flags, _ptr(V), _ptr(pi),
                            _ptr(tr), _ptr(ch), ctypes.byref(st))
    _check(s, (OK, NOT_CONVERGED, NONFINITE))
    o = st.outer_iters
    return Solution(V, pi, tr[: o * (m + 1)], s, st, ch[:o])


# ---------------------------------------------------------- free functions
def partition(n, seed, sweep, identity=False):
    """Host-side partition generator: perm[p] = pi_sweep(p) (numpy uint32)."""
    out = np.empty(n, dtype=np.uint32)
    _check(lib().rmb_partition(n, seed, sweep, ORDER_IDENTITY if identity else 0, _ptr(out)))
    return out


def _select_flag(select):
    if select is None:
        return 0
    if select == "replace":
        return SELECT_REPLACE
    if select == "weighted":
        return SELECT_WEIGHTED
    raise ValueError(f"select must be None, 'replace' or 'weighted', got {select!r}")


def select(n, seed, sweep, weights=None):
    """Host-side generator of application `sweep`'s n draws with replacement
    (uniform, or P(s) ~ weights[s] for integer weights >= 1) -- R28-R29."""
    out = np.empty(n, dtype=np.uint32)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.uint32)
    if w is not None and w.shape != (n,):
        raise ValueError("weights must have n entries")
    _check(lib().rmb_select(n, seed, sweep, _ptr(w), _ptr(out)))
    return out


def partition_device(n, seed, sweep, identity=False, stream=None):
    """The solver's device permutation kernel, into a new cuda uint32-as-int32 tensor."""
    import torch
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    _check(lib().rmb_partition_device(n, seed, sweep, ORDER_IDENTITY if identity else 0, _ptr(out),
                                      _stream_ptr(stream)))
    return out


def generate_dense(n, A, seed, kind="random", dtype=None, rows=None, device="cuda", stream=None):
    """Dense instance (gen/rmb_gen.h) generated on device: P [rows][A][n], c [rows][A]."""
    import torch
    dtype = dtype or torch.float32
    s0, s1 = rows if rows is not None else (0, n)
    P = torch.empty((s1 - s0, A, n), dtype=dtype, device=device)
    c = torch.empty((s1 - s0, A), dtype=dtype, device=device)
    code = F32 if dtype == torch.float32 else F64
    _check(lib().rmb_generate_dense({"random": 0, "dyadic": 1}[kind], seed, n, A, s0, s1, code, _ptr(P), _ptr(c),
                                    _stream_ptr(stream)))
    return P, c


def generate_sparse(n, A, K, seed, dtype=None, rows=None, device="cuda", stream=None):
    import torch
    dtype = dtype or torch.float32
    s0, s1 = rows if rows is not None else (0, n)
    nr = (s1 - s0) * A
    rp = torch.empty(nr + 1, dtype=torch.int64, device=device)
    col = torch.empty(nr * K, dtype=torch.int32, device=device)
    val = torch.empty(nr * K, dtype=dtype, device=device)
    c = torch.empty((s1 - s0, A), dtype=dtype, device=device)
    code = F32 if dtype == torch.float32 else F64
    _check(lib().rmb_generate_sparse(seed, n, A, K, s0, s1, code, _ptr(rp), _ptr(col), _ptr(val), _ptr(c),
                                     _stream_ptr(stream)))
    return rp, col, val, c


def generate_grid(N, dtype=None, rows=None, device="cuda", stream=None):
    import torch
    dtype = dtype or torch.float32
    s0, s1 = rows if rows is not None else (0, N * N)
    nr = (s1 - s0) * 4
    rp = torch.empty(nr + 1, dtype=torch.int64, device=device)
    col = torch.empty(nr * 5, dtype=torch.int32, device=device)
    val = torch.empty(nr * 5, dtype=dtype, device=device)
    c = torch.empty((s1 - s0, 4), dtype=dtype, device=device)
    code = F32 if dtype == torch.float32 else F64
    _check(lib().rmb_generate_grid(N, s0, s1, code, _ptr(rp), _ptr(col), _ptr(val), _ptr(c), _stream_ptr(stream)))
    return rp, col, val, c


def version():
    return lib().rmb_version().decode()
