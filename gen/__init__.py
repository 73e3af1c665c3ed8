"""Seeded synthetic MDP instances (host side), built from gen/rmb_gen.h.

This module is shared by specification *and* code between the two sides of
every parity check: the CUDA library generates the same instances on device
from the same header (paper_2110_02901_b200/csrc/gen_kernels.cu).  It holds
none of the method's arithmetic — only the definition of the instance.

Instance recipes (shapes from BASELINE.json configs,
PAPER.md L483-492):
  dense(kind="random"): w ~ U{1..2^24}, P(.|s,a) = w / sum w, c ~ U[0,1)
  dense(kind="dyadic"): quarter-unit masses on <= 4 columns, integer costs
  sparse: K distinct stratified successors per (s,a), weights as dense
  grid:   N x N gridworld, slip 0.7, goal state 0 (cost 0, absorbing)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgen.so")
_lib = None

KIND = {"random": 0, "dyadic": 1}


def build(force: bool = False) -> str:
    src = [os.path.join(_HERE, "gen_host.c")]
    if force or not os.path.exists(_SO) or any(
        os.path.getmtime(s) > os.path.getmtime(_SO) for s in src + [os.path.join(_HERE, "rmb_gen.h")]
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp", "-o", _SO] + src
        )
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, i32, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p
        lib.gen_dense_rows.argtypes = [ctypes.c_int, u64, i64, i32, i64, i64, ctypes.c_int, vp, vp]
        lib.gen_sparse_rows.argtypes = [u64, i64, i32, i32, i64, i64, ctypes.c_int, vp, vp, vp, vp]
        lib.gen_grid_rows.argtypes = [i64, i64, i64, ctypes.c_int, vp, vp, vp, vp]
        for f in (lib.gen_dense_rows, lib.gen_sparse_rows, lib.gen_grid_rows):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def dense(n: int, A: int, seed: int, kind: str = "random", dtype=np.float32, rows=None):
    """P[s0:s1][A][n] and c[s0:s1][A] of the dense instance (rows=(s0,s1) or all)."""
    s0, s1 = rows if rows is not None else (0, n)
    dtype = np.dtype(dtype)
    P = np.empty((s1 - s0, A, n), dtype=dtype)
    c = np.empty((s1 - s0, A), dtype=dtype)
    rc = _load().gen_dense_rows(KIND[kind], seed, n, A, s0, s1, int(dtype == np.float32), _ptr(P), _ptr(c))
    if rc:
        raise ValueError("gen_dense_rows: bad arguments")
    return P, c


def sparse(n: int, A: int, K: int, seed: int, dtype=np.float32, rows=None):
    """Fixed-width CSR (ELL) of the sparse random instance: row_ptr, col, val, c."""
    s0, s1 = rows if rows is not None else (0, n)
    dtype = np.dtype(dtype)
    nr = (s1 - s0) * A
    row_ptr = np.empty(nr + 1, dtype=np.int64)
    col = np.empty(nr * K, dtype=np.int32)
    val = np.empty(nr * K, dtype=dtype)
    c = np.empty((s1 - s0, A), dtype=dtype)
    rc = _load().gen_sparse_rows(seed, n, A, K, s0, s1, int(dtype == np.float32),
                                 _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(c))
    if rc:
        raise ValueError("gen_sparse_rows: bad arguments")
    return row_ptr, col, val, c


GRID_W = 5


def grid(N: int, dtype=np.float32, rows=None):
    """ELL (width 5) of the N x N slip gridworld: row_ptr, col, val, c (A = 4)."""
    n = N * N
    s0, s1 = rows if rows is not None else (0, n)
    dtype = np.dtype(dtype)
    nr = (s1 - s0) * 4
    row_ptr = np.empty(nr + 1, dtype=np.int64)
    col = np.empty(nr * GRID_W, dtype=np.int32)
    val = np.empty(nr * GRID_W, dtype=dtype)
    c = np.empty((s1 - s0, 4), dtype=dtype)
    rc = _load().gen_grid_rows(N, s0, s1, int(dtype == np.float32), _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(c))
    if rc:
        raise ValueError("gen_grid_rows: bad arguments")
    return row_ptr, col, val, c
