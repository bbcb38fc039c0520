#!/usr/bin/env python
"""Setup-only driver for launch lists: generates the config's matrix in HBM, runs
setup_hierarchy_device `warm` times, then once more (the profiled one).  Prints the library's
kernel-launch count before and during the last setup (ncu --launch-skip / --launch-count)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = sys.argv[2] if len(sys.argv) > 2 else "poisson"
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
lib = M.b200().lib
assert lib.fn("init")(0) == 0
dm = C.c_void_p()
if kind == "jump27":
    assert lib.fn("dmatrix_jump27")(n, n, n, 1e6, 32, C.byref(dm)) == 0
else:
    assert lib.fn("dmatrix_poisson")(3, n, n, n, 1e-3 if kind == "aniso" else 1.0, -1, C.byref(dm)) == 0
s = M.SetupConfig(alpha=0.5, reuse_caches=True)._c()
for i in range(warm + 1):
    before = lib.fn("kernel_launches")()
    h = C.c_void_p()
    assert lib.fn("setup_hierarchy_device")(dm, C.byref(s), C.byref(h)) == 0
    lib.fn("synchronize")()
    after = lib.fn("kernel_launches")()
    ms = C.c_double()
    lib.fn("hierarchy_setup_ms")(h, C.byref(ms))
    lib.fn("hierarchy_free")(h)
    lib.fn("synchronize")()
print(f"LAUNCH_SKIP={before} LAUNCH_COUNT={after - before} SETUP_MS={ms.value:.3f}")
