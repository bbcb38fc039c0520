#!/usr/bin/env python
"""Where the end-to-end (host CSR in, x out) time goes: upload, setup, solve, download."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402


def main(n=256):
    gpu = M.b200()
    lib = gpu.lib
    assert lib.fn("init")(0) == 0
    A = gpu.generate_poisson(3, n, n, n)
    b = np.ones(A.n_rows)
    setup = M.SetupConfig(alpha=0.5, reuse_caches=True)
    solver = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=500)
    gpu.setup_and_solve(A, b, setup, M.CycleConfig(), solver)
    for _ in range(5):
        ca = A._c()
        t0 = time.perf_counter()
        dm = C.c_void_p()
        assert lib.fn("dmatrix_from_host")(C.byref(ca), C.byref(dm)) == 0
        lib.fn("synchronize")()
        t1 = time.perf_counter()
        lib.fn("dmatrix_free")(dm)
        t2 = time.perf_counter()
        res = gpu.setup_and_solve(A, b, setup, M.CycleConfig(), solver)
        t3 = time.perf_counter()
        print(f"upload {1e3*(t1-t0):.1f} ms ({(A.row_offsets.nbytes+A.col_indices.nbytes+A.values.nbytes)/1e9/(t1-t0):.1f} GB/s); "
              f"setup_and_solve {1e3*(t3-t2):.1f} ms (setup incl. upload {1e3*res.report.setup_seconds:.1f}, "
              f"solve {1e3*res.report.solve_seconds:.1f})", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 256)
