#!/usr/bin/env python
"""Setup + solve of a generated problem on the device; prints the residual history as exact
hex floats (compare two builds / switches bit for bit) and the step time."""
import ctypes as C
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import _abi  # noqa: E402
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
kind = sys.argv[2] if len(sys.argv) > 2 else "poisson"
cycle = sys.argv[3] if len(sys.argv) > 3 else "hybrid"
lib = M.b200().lib
assert lib.fn("init")(0) == 0
dm = C.c_void_p()
if kind == "jump27":
    assert lib.fn("dmatrix_jump27")(n, n, n, 1e6, 32, C.byref(dm)) == 0
else:
    assert lib.fn("dmatrix_poisson")(3, n, n, n, 1e-3 if kind == "aniso" else 1.0, -1, C.byref(dm)) == 0
s = M.SetupConfig(alpha=0.5, reuse_caches=True)._c()
c = M.CycleConfig(kind={"v": M.CYCLE_V, "k": M.CYCLE_K, "hybrid": M.CYCLE_HYBRID}[cycle])._c()
v = M.SolverConfig(method=M.FGMRES if kind == "aniso" else M.PCG, tol=1e-8, max_iters=500,
                   restart=30)._c()
hist = np.zeros(600)
x = np.zeros(n ** 3)
for step in range(3):
    h = C.c_void_p()
    lib.fn("synchronize")()
    ts = time.perf_counter()
    assert lib.fn("setup_hierarchy_device")(dm, C.byref(s), C.byref(h)) == 0
    lib.fn("synchronize")()
    setup_ms = 1e3 * (time.perf_counter() - ts)
    rep = _abi.SolveReportC()
    rep.history = hist.ctypes.data_as(_abi.f64p)
    rep.history_capacity = 600
    lib.fn("synchronize")()
    t0 = time.perf_counter()
    assert lib.fn("solve_device")(h, C.byref(c), C.byref(v), x.ctypes.data_as(_abi.f64p),
                                  C.byref(rep)) == 0, lib.fn("last_error")()
    lib.fn("synchronize")()
    dt = time.perf_counter() - t0
    lib.fn("hierarchy_free")(h)
hh = hist[: rep.history_length]
print(f"its={rep.iterations} setup_ms={setup_ms:.2f} solve_ms={1e3 * dt:.2f} history_sha={hashlib.sha256(hh.tobytes()).hexdigest()[:16]} "
      f"x_sha={hashlib.sha256(x.tobytes()).hexdigest()[:16]}")
