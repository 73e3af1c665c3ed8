"""Build librmb.so (sm_100a) in-tree with nvcc."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "librmb.so")
BUILD = os.path.join(HERE, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_include():
    """nccl.h for the NCCL types (the library itself is dlopen'ed at run time)."""
    cands = []
    try:
        import nvidia.nccl  # torch's NCCL wheel
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands += ["/usr/include", "/usr/local/cuda/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


NVFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                  "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", _nccl_include()]


def _nvcc():
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps():
    return (glob.glob(os.path.join(CSRC, "*")) + [os.path.join(ROOT, "include", "rmb.h"),
                                                  os.path.join(ROOT, "gen", "rmb_gen.h")])


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """out/defines: alternative builds for A/B experiments (never the product .so)."""
    so = out or SO
    if not force and out is None and not needs_build():
        return SO
    bdir = BUILD if out is None else BUILD + "_" + os.path.basename(out).replace(".so", "")
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    dflags = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        r = subprocess.run([nvcc] + NVFLAGS + dflags + ["-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = so + ".tmp"
    r = subprocess.run([nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, so)
    if verbose:
        for o in objs:
            print(open(o + ".ptxas.txt").read())
    return so


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(SO)
