#!/usr/bin/env python
"""SGS-smoothed hierarchies (SetupConfig.smoother = sgs): setup + solve time on the GPU
(level-scheduled sweeps) beside the reference on the host cores (oracle/_ref), same
iterations.  Usage: sgs_bench.py [2d_n] [3d_n]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402
from oracle import checkers  # noqa: E402


def run(impl, A, alpha, reps):
    cfg = M.SetupConfig(alpha=alpha, reuse_caches=True, smoother=M.SGS)
    sc = M.SolverConfig(method=M.FGMRES, tol=1e-8, max_iters=500, restart=30)
    b = np.ones(A.n_rows)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        h = impl.setup_hierarchy(A, None, cfg)
        t1 = time.perf_counter()
        r = impl.fgmres(A, b, None, h, None, sc)
        t2 = time.perf_counter()
        cur = (t1 - t0, t2 - t1, r.report.iterations)
        best = cur if best is None or cur[0] + cur[1] < best[0] + best[1] else best
    return best


def main():
    n2 = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    n3 = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    gpu, ref = M.b200(), checkers.ref()
    assert gpu.lib.fn("init")(0) == 0
    for name, A, alpha in ((f"2d {n2}^2", gpu.generate_poisson(2, n2, n2), 0.25),
                           (f"3d {n3}^3", gpu.generate_poisson(3, n3, n3, n3), 0.5)):
        g = run(gpu, A, alpha, 3)
        r = run(ref, A, alpha, 1)
        print(f"{name}: gpu setup {1e3*g[0]:.1f} ms solve {1e3*g[1]:.1f} ms ({g[2]} its) | "
              f"ref setup {1e3*r[0]:.1f} ms solve {1e3*r[1]:.1f} ms ({r[2]} its)", flush=True)


if __name__ == "__main__":
    main()
