"""A/B library builds: one source file of csrc/ recompiled with extra -D
defines and linked with the product build's other objects.

  from tools.ab_build import build_variants
  build_variants("dense.cu", {"name": ["MACRO=1", ...], ...})  -> {name: path}
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lib_path(name):
    return os.path.join(ROOT, "build_ab", f"librmb_{name}.so")


def build_variants(src, variants):
    from paper_2110_02901_b200 import _build
    _build.build()
    os.makedirs(os.path.join(ROOT, "build_ab"), exist_ok=True)
    nvcc = _build._nvcc()
    others = [os.path.join(_build.BUILD, f) for f in sorted(os.listdir(_build.BUILD))
              if f.endswith(".cu.o") and f != src + ".o"]

    def one(item):
        name, d = item
        obj = os.path.join(ROOT, "build_ab", f"{src}_{name}.o")
        with open(obj + ".ptxas.txt", "w") as log:
            subprocess.check_call([nvcc] + _build.NVFLAGS + [f"-D{x}" for x in d] +
                                  ["-c", os.path.join(_build.CSRC, src), "-o", obj], stderr=log)
        subprocess.check_call([nvcc] + _build.ARCH + ["-shared", "-o", lib_path(name), obj] + others + ["-ldl"])
        return name, lib_path(name)

    with ThreadPoolExecutor(len(variants)) as ex:
        return dict(ex.map(one, variants.items()))
