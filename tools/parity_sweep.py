#!/usr/bin/env python
"""Randomised parity sweep against the reference (oracle/_ref): hierarchies bit-identical
(cache path), preconditioner applications within 1e-12, PCG / FGMRES iteration counts equal
with histories within 1e-10 * ||r0||.  Problems: 2-D / 3-D Poisson with random sizes and
anisotropy, 27-point jump operators, random SPD matrices; random smoother / cycle / solver
settings, and a large class past the SELL-32 threshold (>= 2^19 rows: level 0 in SELL-32, with
the value dictionary on stencils, plain on variable coefficients).
Usage: parity_sweep.py [seconds] [seed] [exact|default] [large]
exact: aggmg_set_exact_reductions(1) for the whole sweep, and the bar becomes bit-identical
residual histories and solutions; large: only the >= 2^19-row class.
History bar (default mode): |h_k - h_k^ref| <= 1e-10 * max_j h_j^ref."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402
from oracle import checkers  # noqa: E402
from helpers import bits, random_spd  # noqa: E402
from test_gpu_parity_sell import variable_poisson3d  # noqa: E402


def large_problem(gpu, rng):
    """>= 2^19 rows: the SELL-32 kernels (and the value dictionary on stencils) at level 0."""
    kind = rng.integers(0, 3)
    if kind == 0:
        nx, ny, nz = rng.integers(80, 129, 3)
        eps = float(rng.choice([1.0, 1.0, 1e-3]))
        return f"L 3d {nx}x{ny}x{nz} eps={eps}", gpu.generate_poisson(3, int(nx), int(ny), int(nz), eps), 0.5
    if kind == 1:
        nx, ny, nz = rng.integers(81, 100, 3)
        blk = int(rng.choice([8, 16, 32]))
        return f"L jump27 {nx}x{ny}x{nz}/{blk}", gpu.generate_jump27(int(nx), int(ny), int(nz), 1e6, blk), 0.5
    n = int(rng.integers(81, 100))
    return f"L variable3d {n}", variable_poisson3d(n, int(rng.integers(0, 1 << 30))), 0.5


def problem(gpu, rng, large_only=False):
    if large_only or rng.random() < 0.12:
        return large_problem(gpu, rng)
    kind = rng.integers(0, 4)
    if kind == 0:
        nx, ny = rng.integers(8, 160, 2)
        eps = float(rng.choice([1.0, 0.1, 1e-3]))
        return f"2d {nx}x{ny} eps={eps}", gpu.generate_poisson(2, int(nx), int(ny), 1, eps), 0.25
    if kind == 1:
        nx, ny, nz = rng.integers(6, 40, 3)
        eps = float(rng.choice([1.0, 1e-3]))
        return f"3d {nx}x{ny}x{nz} eps={eps}", gpu.generate_poisson(3, int(nx), int(ny), int(nz), eps), 0.5
    if kind == 2:
        nx, ny, nz = rng.integers(5, 24, 3)
        blk = int(rng.integers(2, 6))
        return f"jump27 {nx}x{ny}x{nz}/{blk}", gpu.generate_jump27(int(nx), int(ny), int(nz), 1e6, blk), 0.5
    n = int(rng.integers(50, 1500))
    return f"spd {n}", random_spd(n, float(rng.uniform(0.002, 0.05)), int(rng.integers(0, 1 << 30))), 0.25


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    gpu, ref = M.b200(), checkers.ref()
    assert gpu.lib.fn("init")(0) == 0
    exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
    large_only = len(sys.argv) > 4 and sys.argv[4] == "large"
    big = 0
    if exact:
        gpu.lib.fn("set_exact_reductions")(1)
    t0, count, fails = time.time(), 0, 0
    while time.time() - t0 < budget:
        name, A, alpha = problem(gpu, rng, large_only)
        big += A.n_rows >= (1 << 19)
        smoother = int(rng.choice([M.JACOBI, M.DAMPED_JACOBI, M.DAMPED_JACOBI, M.SGS]))
        cfg = M.SetupConfig(alpha=alpha, reuse_caches=True, smoother=smoother,
                            coarse_size_max=int(rng.choice([20, 60, 600])))
        cyc = M.CycleConfig(kind=int(rng.choice([M.CYCLE_V, M.CYCLE_K, M.CYCLE_HYBRID])),
                            inner=int(rng.choice([M.INNER_CG, M.INNER_GMRES])),
                            t=float(rng.choice([0.0, 0.25, 1e9])))
        tag = f"{name} smoother={smoother} cyc=({cyc.kind},{cyc.inner},{cyc.t}) cmax={cfg.coarse_size_max}"
        try:
            hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
            assert hg.n_levels() == hr.n_levels(), "levels"
            for k in range(hg.n_levels()):
                a, b = hg.levels[k].A, hr.levels[k].A
                assert np.array_equal(a.col_indices, b.col_indices), f"L{k} pattern"
                assert np.array_equal(bits(a.values), bits(b.values)), f"L{k} values"
            r = rng.uniform(-1, 1, A.n_rows)
            zg, zr = gpu.apply_preconditioner(hg, cyc, r), ref.apply_preconditioner(hr, cyc, r)
            rel = np.linalg.norm(zg - zr) / max(np.linalg.norm(zr), 1e-300)
            assert rel <= 1e-12, f"preconditioner rel {rel:.2e}"
            method = M.FGMRES if smoother == M.SGS or rng.random() < 0.5 else M.PCG
            sc = M.SolverConfig(method=method, tol=1e-8, max_iters=300, restart=int(rng.choice([10, 30])))
            bvec = np.ones(A.n_rows)
            f = gpu.pcg if method == M.PCG else gpu.fgmres
            g = ref.pcg if method == M.PCG else ref.fgmres
            rg, rr = f(A, bvec, None, hg, cyc, sc), g(A, bvec, None, hr, cyc, sc)
            assert rg.report.iterations == rr.report.iterations, \
                f"iterations {rg.report.iterations} vs {rr.report.iterations}"
            hg_, hr_ = np.array(rg.report.residual_history), np.array(rr.report.residual_history)
            if exact:
                assert hg_.shape == hr_.shape and np.array_equal(bits(hg_), bits(hr_)), "exact history"
                assert np.array_equal(bits(rg.x), bits(rr.x)), "exact x"
                count += 1
                continue
            dev = np.max(np.abs(hg_ - hr_)) / np.max(hr_)
            if dev > 1e-10:
                # rounding-order sensitivity or a real difference?  rerun with the reference's
                # 8192-chunk reduction order on the device
                gpu.lib.fn("set_exact_reductions")(1)
                try:
                    re_ = f(A, bvec, None, hg, cyc, sc)
                finally:
                    gpu.lib.fn("set_exact_reductions")(0)
                he = np.array(re_.report.residual_history)
                dev_e = (np.max(np.abs(he - hr_)) / np.max(hr_)) if he.shape == hr_.shape else float("inf")
                raise AssertionError(f"history {dev:.2e} (method {method}, its {rg.report.iterations}); "
                                     f"exact-order rerun {dev_e:.2e}")
        except M.Error as e:  # the same error on both sides is parity too
            try:
                ref.setup_hierarchy(A, None, cfg)
                print(f"FAIL {tag}: gpu error only: {e}", flush=True)
                fails += 1
            except M.Error as e2:
                if str(e).split(":")[0] != str(e2).split(":")[0]:
                    print(f"FAIL {tag}: errors differ: {e} / {e2}", flush=True)
                    fails += 1
        except AssertionError as e:
            print(f"FAIL {tag}: {e}", flush=True)
            fails += 1
        count += 1
    print(f"parity sweep ({'exact' if exact else 'default'} mode): {count} cases ({big} with >= 2^19 rows), "
          f"{fails} failures, {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
