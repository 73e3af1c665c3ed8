"""A/B of the asynchronous dense kernel's CTA shape on config 2: ms per
asynchronous application (30 applications, V0 = 0), per library build.

  python tools/ab_async.py build      # (CPU) the variant libraries
  python tools/ab_async.py run        # (GPU) one subprocess per variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {"nt512": ["RMB_ASYNC_NT=512"], "nt256": ["RMB_ASYNC_NT=256"], "nt128": ["RMB_ASYNC_NT=128"],
            "nt64": ["RMB_ASYNC_NT=64"]}
if len(sys.argv) > 2:
    VARIANTS = {k: v for k, v in VARIANTS.items() if k in sys.argv[2].split(",")}


def lib_of(name):
    return os.path.join(ROOT, "build_ab", f"librmb_{name}.so")


def build():
    """Only async.cu differs: compile it per variant, link with the product build's other objects."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2110_02901_b200 import _build
    _build.build()
    os.makedirs(os.path.join(ROOT, "build_ab"), exist_ok=True)
    nvcc = _build._nvcc()
    others = [os.path.join(_build.BUILD, f) for f in sorted(os.listdir(_build.BUILD))
              if f.endswith(".cu.o") and f != "async.cu.o"]

    def one_variant(item):
        name, d = item
        obj = os.path.join(ROOT, "build_ab", f"async_{name}.o")
        subprocess.check_call([nvcc] + _build.NVFLAGS + [f"-D{x}" for x in d] +
                              ["-c", os.path.join(_build.CSRC, "async.cu"), "-o", obj],
                              stderr=open(obj + ".ptxas.txt", "w"))
        subprocess.check_call([nvcc] + _build.ARCH + ["-shared", "-o", lib_of(name), obj] + others + ["-ldl"])

    with ThreadPoolExecutor(len(VARIANTS)) as ex:
        list(ex.map(one_variant, VARIANTS.items()))


def one():
    import torch
    import paper_2110_02901_b200 as rmb
    n, A = 10_000, 16
    P, c = rmb.generate_dense(n, A, 1)
    prob = rmb.Problem.dense(P, c, 0.99, flags=rmb.DENSE_NO_TMA if os.environ.get("AB_ASYNC_REGS") else 0)
    prob.vi(1, eps=1e-6, max_sweeps=3, asynchronous=True)
    best = 1e9
    for rep in range(3):
        sol = prob.vi(1, seed=rep, eps=1e-9, max_sweeps=30, asynchronous=True)
        best = min(best, sol.stats.seconds / sol.stats.sweeps)
    sol = prob.vi(1, seed=0, eps=1e-6, max_sweeps=100_000, asynchronous=True)
    print(json.dumps({"lib": os.environ.get("RMB_LIB_PATH"), "ms_per_app": best * 1e3,
                      "GB_per_s": 6.4e9 / best / 1e9, "sweeps_to_eps": sol.stats.sweeps,
                      "time_to_eps_ms": sol.stats.seconds * 1e3}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    elif sys.argv[1] == "one":
        one()
    else:
        for name in VARIANTS:
            env = dict(os.environ, RMB_LIB_PATH=lib_of(name), AB_ASYNC_REGS="1")
            subprocess.run([sys.executable, __file__, "one"], env=env, check=False)
