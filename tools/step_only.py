#!/usr/bin/env python
"""One bench step (setup_hierarchy_device + solve_device) after `warm` warm-up steps, for
launch lists: prints the library's launch count before and during the last step (ncu
--launch-skip / --launch-count), so matrix generation and warm-up are excluded."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import _abi  # noqa: E402
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
c = M.CycleConfig()._c()
v = M.SolverConfig(method=M.FGMRES if kind == "aniso" else M.PCG, tol=1e-8, max_iters=500,
                   restart=30)._c()
hist = np.zeros(600)
for i in range(warm + 1):
    before = lib.fn("kernel_launches")()
    h = C.c_void_p()
    assert lib.fn("setup_hierarchy_device")(dm, C.byref(s), C.byref(h)) == 0
    mid = lib.fn("kernel_launches")()
    rep = _abi.SolveReportC()
    rep.history = hist.ctypes.data_as(_abi.f64p)
    rep.history_capacity = 600
    assert lib.fn("solve_device")(h, C.byref(c), C.byref(v), None, C.byref(rep)) == 0
    lib.fn("synchronize")()
    after = lib.fn("kernel_launches")()
    lib.fn("hierarchy_free")(h)
print(f"LAUNCH_SKIP={before} LAUNCH_COUNT={after - before} SETUP_LAUNCHES={mid - before} "
      f"ITERATIONS={rep.iterations}")
