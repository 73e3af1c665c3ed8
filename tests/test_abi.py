"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/*.h declares, and its host-side pieces (partition generator, argument
checks, status strings) behave — no GPU needed."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import oracle
import paper_2110_02901_b200 as rmb
from conftest import ROOT


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(rmb_[a-z_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(rmb.LIB_PATH)
    decl = declared_functions()
    assert len(decl) >= 15
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    # and the binding marshals every one of them
    assert sorted(rmb.exported_symbols()) == decl


def test_status_strings_and_version():
    L = rmb.lib()
    assert L.rmb_status_string(0) == b"RMB_OK"
    assert L.rmb_status_string(8) == b"RMB_ERR_UNSUPPORTED"
    assert rmb.version().startswith("rmb")


@pytest.mark.parametrize("n,seed,k", [(1, 0, 1), (2, 5, 3), (50, 42, 7), (1000, 9, 1), (10_000, 3, 11),
                                      (1_000_000, 123, 2)])
def test_host_partition_generator_matches_oracle(n, seed, k):
    # two independent implementations of SURVEY 8(c)-1 (library C++ vs oracle C)
    assert np.array_equal(rmb.partition(n, seed, k), oracle.partition(n, seed, k))


def test_host_partition_identity():
    assert np.array_equal(rmb.partition(9, 1, 1, identity=True), np.arange(9))


def test_argument_errors_before_device_work():
    L = rmb.lib()
    d = rmb._Desc(10, 2, 1.5, rmb.F32, rmb.F64, 0, 10, None, None)   # gamma out of (0,1)
    h = ctypes.c_void_p()
    buf = np.zeros(200, np.float32)
    st = L.rmb_create_dense(ctypes.byref(d), buf.ctypes.data, buf.ctypes.data, 0, ctypes.byref(h))
    assert st == rmb.INVALID_ARG and b"gamma" in L.rmb_last_error()
    d = rmb._Desc(10, 2, 0.9, rmb.F32, rmb.F32, 0, 10, None, None)   # fp32 V unsupported
    assert L.rmb_create_dense(ctypes.byref(d), buf.ctypes.data, buf.ctypes.data, 0, ctypes.byref(h)) == rmb.INVALID_ARG
    assert L.rmb_partition(0, 0, 1, 0, None) == rmb.INVALID_ARG
    assert L.rmb_vi(None, 1, 0, 1e-6, 10, 0, None, None, None, None) == rmb.INVALID_ARG


@pytest.mark.parametrize("n,seed,k", [(1, 0, 1), (17, 3, 2), (1000, 9, 5), (65_537, 2**40 + 1, 77)])
@pytest.mark.parametrize("weighted", [False, True])
def test_host_select_matches_oracle(n, seed, k, weighted):
    """The product's host draw generator (partition.cuh Selection, R28-R29) is
    bitwise the oracle's independent implementation."""
    import oracle
    w = np.random.default_rng(n).integers(1, 2**32, size=n, dtype=np.uint64).astype(np.uint32) if weighted else None
    assert np.array_equal(rmb.select(n, seed, k, w), oracle.select(n, seed, k, w))


def test_host_select_rejects_zero_weight():
    with pytest.raises(rmb.RmbError):
        rmb.select(3, 1, 1, np.array([1, 0, 2], np.uint32))
