"""A/B of the asynchronous TMA kernel's stage geometry (slot KB, rows per unit)
on config 2: ms per asynchronous application.  build (CPU) / run (GPU)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.ab_build import build_variants, lib_path  # noqa: E402

VARIANTS = {"rw4_s72": ["RMB_TA_RW=4", "RMB_TA_SLOT_KB=72"], "rw4_s56": ["RMB_TA_RW=4", "RMB_TA_SLOT_KB=56"],
            "rw8_s72": ["RMB_TA_RW=8", "RMB_TA_SLOT_KB=72"], "rw16_s72": ["RMB_TA_RW=16", "RMB_TA_SLOT_KB=72"],
            "rw4_c14_s72": ["RMB_TA_RW=4", "RMB_TA_CONS=14", "RMB_TA_SLOT_KB=72"],
            "rw4_s104": ["RMB_TA_RW=4", "RMB_TA_SLOT_KB=104"]}

if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_variants("async.cu", VARIANTS)
    else:
        for name in VARIANTS:
            subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ab_async.py"), "one"],
                           env=dict(os.environ, RMB_LIB_PATH=lib_path(name)))
