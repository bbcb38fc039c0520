#!/usr/bin/env python
"""Wall-clock split of one bench step (setup / solve / free) on the device path."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import _abi  # noqa: E402
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
kind = sys.argv[2] if len(sys.argv) > 2 else "poisson"
lib = M.b200().lib
assert lib.fn("init")(0) == 0
dm = C.c_void_p()
if kind == "jump27":
    assert lib.fn("dmatrix_jump27")(n, n, n, 1e6, 32, C.byref(dm)) == 0
elif kind == "aniso":  # c3: eps = 1e-3 on z, FGMRES(30)
    assert lib.fn("dmatrix_poisson")(3, n, n, n, 1e-3, -1, C.byref(dm)) == 0
else:
    assert lib.fn("dmatrix_poisson")(3, n, n, n, 1.0, -1, C.byref(dm)) == 0
s = M.SetupConfig(alpha=0.5, reuse_caches=True)._c()
c = M.CycleConfig()._c()
v = M.SolverConfig(method=M.FGMRES if kind == "aniso" else M.PCG, tol=1e-8, max_iters=500,
                   restart=30)._c()
hist = np.zeros(600)
if os.environ.get("EXACT"):  # aggmg_set_exact_reductions(1): the bit-identical mode
    lib.fn("set_exact_reductions")(1)
prof = None
if os.environ.get("KERNELS"):  # CUPTI kernel table of the last step (torch.profiler)
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.init()
steps = int(os.environ.get("STEPS", "4"))
for step in range(steps):
    if os.environ.get("KERNELS") and step == steps - 1:
        prof = profile(activities=[ProfilerActivity.CUDA])
        prof.__enter__()
    t0 = time.perf_counter()
    h = C.c_void_p()
    assert lib.fn("setup_hierarchy_device")(dm, C.byref(s), C.byref(h)) == 0
    lib.fn("synchronize")()
    t1 = time.perf_counter()
    rep = _abi.SolveReportC()
    rep.history = hist.ctypes.data_as(_abi.f64p)
    rep.history_capacity = 600
    assert lib.fn("solve_device")(h, C.byref(c), C.byref(v), None, C.byref(rep)) == 0
    lib.fn("synchronize")()
    t2 = time.perf_counter()
    lib.fn("hierarchy_free")(h)
    lib.fn("synchronize")()
    t3 = time.perf_counter()
    print(f"step {step}: setup {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms ({rep.iterations} its), "
          f"free {1e3*(t3-t2):.1f} ms; report: solve {1e3*rep.solve_seconds:.1f} ms", flush=True)
if prof is not None:
    prof.__exit__(None, None, None)
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
