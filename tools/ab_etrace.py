"""A/B: the dense solver with / without the error-trace call compiled in
(config 2 ms per sweep at b = 1000 and b = n).  build (CPU) / run (GPU)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.ab_build import build_variants, lib_path  # noqa: E402

VARIANTS = {"etrace": [], "noetrace": ["RMB_AB_NO_ETRACE=1"]}

if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_variants("dense.cu", VARIANTS)
    else:
        for rep in range(2):
            for name in VARIANTS:
                print(name, flush=True)
                subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ab_tma.py"), "10000,1000,64"],
                               env=dict(os.environ, RMB_LIB_PATH=lib_path(name)))
