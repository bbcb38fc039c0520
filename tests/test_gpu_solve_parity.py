"""Solve-stage parity against the unmodified reference (oracle/_ref).  SpMV / smoothers /
restriction / prolongation are bit-exact (row-sequential sums, no FMA); cycles and
Krylov histories agree within 1e-10 relative (only dot-product summation order differs,
SURVEY §8a rows a14-a20); outer iteration counts are equal."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import bits, laplacian_1d, max_rel, random_sparse, random_spd, rel_norm

pytestmark = pytest.mark.gpu


def test_spmv_bit_exact(gpu, ref):
    rng = np.random.default_rng(0)
    mats = [ref.generate_poisson(2, 33, 31), ref.generate_poisson(3, 17, 9, 11, 0.1),
            random_sparse(300, 200, 0.05, 3), random_spd(257, 0.2, 5), laplacian_1d(1000),
            random_sparse(50, 50, 0.9, 8), gpu.generate_jump27(9, 8, 7, 1e6, 2)]
    for A in mats:
        x = rng.uniform(-1, 1, A.n_cols)
        np.testing.assert_array_equal(bits(gpu.spmv(A, x)), bits(ref.spmv(A, x)))


def test_spmv_long_rows(gpu, ref):
    # rows longer than one staging block (dense-ish rows of a coarse operator)
    A = random_sparse(40, 9000, 0.6, 2)
    x = np.random.default_rng(1).uniform(-1, 1, 9000)
    np.testing.assert_array_equal(bits(gpu.spmv(A, x)), bits(ref.spmv(A, x)))


def test_transpose(gpu, ref):
    for s in range(3):
        A = random_sparse(120, 90, 0.07, s)
        T1, T2 = gpu.transpose(A), ref.transpose(A)
        np.testing.assert_array_equal(T1.row_offsets, T2.row_offsets)
        np.testing.assert_array_equal(T1.col_indices, T2.col_indices)
        np.testing.assert_array_equal(bits(T1.values), bits(T2.values))


def test_vector_ops(gpu, ref):
    rng = np.random.default_rng(2)
    for n in (1, 1000, 100_003):
        a, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        # aggmg_dot / aggmg_norm2 use the reference's 8192-chunk order: bit-identical
        assert gpu.dot(a, b) == ref.dot(a, b)
        assert gpu.norm2(a) == ref.norm2(a)
        np.testing.assert_array_equal(bits(gpu.axpy(0.3, a, b)), bits(ref.axpy(0.3, a, b)))
        np.testing.assert_array_equal(bits(gpu.scale(-1.7, a)), bits(ref.scale(-1.7, a)))


def test_smoothers_bit_exact(gpu, ref):
    rng = np.random.default_rng(4)
    A = ref.generate_poisson(2, 20, 20)
    s = ref.setup_smoother(A, M.DAMPED_JACOBI, 5, 9)
    b, x = rng.uniform(-1, 1, A.n_rows), rng.uniform(-1, 1, A.n_rows)
    for kind in (M.JACOBI, M.DAMPED_JACOBI, M.SGS):
        st = M.SmootherState(kind, s.inv_diag, s.omega, s.rho_est)
        np.testing.assert_array_equal(bits(gpu.smooth(st, A, b, x)), bits(ref.smooth(st, A, b, x)))


def _with_diag(A, seed):
    """random nonsymmetric pattern plus a dominant diagonal (sgs needs 1/A_ii)"""
    from helpers import from_triplets
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    rows = np.concatenate([r, np.arange(A.n_rows)])
    cols = np.concatenate([A.col_indices, np.arange(A.n_rows)])
    vals = np.concatenate([A.values, rng.uniform(4, 5, A.n_rows)])
    return from_triplets(A.n_rows, A.n_cols, rows, cols, vals)


def test_sgs_level_schedule_bit_exact(gpu, ref):
    # the level-scheduled sweep against the reference's sequential one: narrow levels (2-D,
    # 1-D chain), wide levels (3-D 40^3: planes of up to ~2,400 rows), long rows (27-point),
    # nonsymmetric patterns (rows read columns whose rows do not read them back)
    rng = np.random.default_rng(11)
    mats = [ref.generate_poisson(2, 20, 20), ref.generate_poisson(3, 40, 40, 40),
            ref.generate_poisson(3, 30, 20, 10, 1e-3), laplacian_1d(3000), random_spd(300, 0.1, 2),
            _with_diag(random_sparse(500, 500, 0.01, 4), 5), gpu.generate_jump27(14, 13, 12, 1e6, 3)]
    for A in mats:
        s = ref.setup_smoother(A, M.JACOBI, 5, 0)
        st = M.SmootherState(M.SGS, s.inv_diag, 1.0, 1.0)
        b, x = rng.uniform(-1, 1, A.n_rows), rng.uniform(-1, 1, A.n_rows)
        np.testing.assert_array_equal(bits(gpu.smooth(st, A, b, x)), bits(ref.smooth(st, A, b, x)))


@pytest.mark.parametrize("ci", [0, 1, 2])
def test_sgs_hierarchy_preconditioner(gpu, ref, ci):
    A = ref.generate_poisson(2, 60, 60)
    cfg = M.SetupConfig(coarse_size_max=40, reuse_caches=True, smoother=M.SGS)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    r = np.random.default_rng(5).uniform(-1, 1, A.n_rows)
    zg, zr = gpu.apply_preconditioner(hg, CFGS[ci], r), ref.apply_preconditioner(hr, CFGS[ci], r)
    assert rel_norm(zg, zr) <= 1e-12


def test_sgs_fgmres(gpu, ref):
    A = ref.generate_poisson(3, 24, 24, 24)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, smoother=M.SGS)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    sc = M.SolverConfig(method=M.FGMRES, tol=1e-8, max_iters=200, restart=30)
    b = np.ones(A.n_rows)
    rg, rr = gpu.fgmres(A, b, None, hg, None, sc), ref.fgmres(A, b, None, hr, None, sc)
    assert rg.report.iterations == rr.report.iterations
    assert hist_close(rg.report.residual_history, rr.report.residual_history)
    assert rel_norm(rg.x, rr.x) <= 1e-10


CFGS = [M.CycleConfig(), M.CycleConfig(kind=M.CYCLE_V), M.CycleConfig(kind=M.CYCLE_K),
        M.CycleConfig(inner=M.INNER_CG), M.CycleConfig(t=1e9), M.CycleConfig(t=0.0)]


@pytest.mark.parametrize("ci", range(len(CFGS)))
def test_preconditioner_matches(gpu, ref, ci):
    A = ref.generate_poisson(2, 60, 60)
    cfg = M.SetupConfig(coarse_size_max=40, reuse_caches=True)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    r = np.random.default_rng(5).uniform(-1, 1, A.n_rows)
    zg, zr = gpu.apply_preconditioner(hg, CFGS[ci], r), ref.apply_preconditioner(hr, CFGS[ci], r)
    assert rel_norm(zg, zr) <= 1e-12


def test_cycles_nonzero_guess(gpu, ref):
    A = ref.generate_poisson(3, 12, 12, 12)
    cfg = M.SetupConfig(alpha=0.5, coarse_size_max=30, reuse_caches=True)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    rng = np.random.default_rng(6)
    b, x = rng.uniform(-1, 1, A.n_rows), rng.uniform(-1, 1, A.n_rows)
    assert rel_norm(gpu.vcycle(hg, 0, b, x), ref.vcycle(hr, 0, b, x)) <= 1e-12
    cc = M.CycleConfig()
    assert rel_norm(gpu.kcycle(hg, cc, 0, b, x), ref.kcycle(hr, cc, 0, b, x)) <= 1e-12
    n1 = hg.levels[1].n
    b1, x1 = rng.uniform(-1, 1, n1), np.zeros(n1)
    assert rel_norm(gpu.vcycle(hg, 1, b1, x1), ref.vcycle(hr, 1, b1, x1)) <= 1e-12


def check_solve(gpu, ref, A, alpha, method, tol=1e-8, cycle=None, restart=30):
    cfg = M.SetupConfig(alpha=alpha, reuse_caches=True)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    sc = M.SolverConfig(method=method, tol=tol, max_iters=500, restart=restart)
    b = np.ones(A.n_rows)
    f = gpu.pcg if method == M.PCG else gpu.fgmres
    g = ref.pcg if method == M.PCG else ref.fgmres
    rg, rr = f(A, b, None, hg, cycle, sc), g(A, b, None, hr, cycle, sc)
    assert rg.report.iterations == rr.report.iterations
    assert rg.report.converged == rr.report.converged
    assert hist_close(rg.report.residual_history, rr.report.residual_history)
    assert rel_norm(rg.x, rr.x) <= 1e-10
    return rg


def hist_close(hg, hr, tol=1e-10):
    """Residual histories agree within tol relative to the initial residual norm."""
    hg, hr = np.asarray(hg), np.asarray(hr)
    return hg.shape == hr.shape and float(np.max(np.abs(hg - hr))) <= tol * hr[0]


def test_pcg_2d(gpu, ref):
    check_solve(gpu, ref, ref.generate_poisson(2, 128, 128), 0.25, M.PCG)


def test_pcg_3d(gpu, ref):
    check_solve(gpu, ref, ref.generate_poisson(3, 32, 32, 32), 0.5, M.PCG)


def test_fgmres_3d_aniso(gpu, ref):
    check_solve(gpu, ref, ref.generate_poisson(3, 32, 32, 32, 1e-3), 0.5, M.FGMRES)


def test_fgmres_small_restart(gpu, ref):
    check_solve(gpu, ref, ref.generate_poisson(2, 64, 64, 1, 0.01), 0.25, M.FGMRES, 1e-10,
                M.CycleConfig(kind=M.CYCLE_V), restart=5)


def test_unpreconditioned(gpu, ref):
    A = random_spd(200, 0.05, 3)
    b = np.random.default_rng(1).uniform(-1, 1, 200)
    for name in ("pcg", "fgmres"):
        sc = M.SolverConfig(method=M.PCG if name == "pcg" else M.FGMRES, tol=1e-10, max_iters=300,
                            restart=20)
        rg = getattr(gpu, name)(A, b, None, None, None, sc)
        rr = getattr(ref, name)(A, b, None, None, None, sc)
        assert rg.report.iterations == rr.report.iterations
        assert hist_close(rg.report.residual_history, rr.report.residual_history)


def test_pcg_rejects_indefinite(gpu, ref):
    A = M.SparseMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    with pytest.raises(M.Error, match="use fgmres"):
        gpu.pcg(A, np.array([1.0, 1.0]), None, None, None, M.SolverConfig(method=M.PCG))


def test_setup_and_solve(gpu, ref):
    A = ref.generate_poisson(3, 24, 24, 24)
    s = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=500)
    rg = gpu.setup_and_solve(A, np.ones(A.n_rows), s, M.CycleConfig(), sc)
    rr = ref.setup_and_solve(A, np.ones(A.n_rows), s, M.CycleConfig(), sc)
    assert rg.report.iterations == rr.report.iterations
    assert hist_close(rg.report.residual_history, rr.report.residual_history)


def test_refresh_values(gpu, ref):
    A = ref.generate_poisson(2, 40, 40)
    cfg = M.SetupConfig(reuse_caches=True, coarse_size_max=30)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    v = A.values * 2.0
    gpu.refresh_values(hg, v)
    ref.refresh_values(hr, v)
    for k in range(hg.n_levels()):
        np.testing.assert_array_equal(bits(hg.levels[k].A.values), bits(hr.levels[k].A.values))
    h0 = gpu.setup_hierarchy(A, None, M.SetupConfig(coarse_size_max=30))
    with pytest.raises(M.Error, match="without caches"):
        gpu.refresh_values(h0, v)


EXACT_CASES = [
    ("3d-aniso-fgmres", (3, 24, 24, 24, 1e-3), 0.5, M.DAMPED_JACOBI, M.CycleConfig(), M.FGMRES),
    ("2d-pcg", (2, 100, 100, 1, 1.0), 0.25, M.DAMPED_JACOBI, M.CycleConfig(), M.PCG),
    ("2d-aniso-undamped-k", (2, 149, 152, 1, 1e-3), 0.25, M.JACOBI,
     M.CycleConfig(kind=M.CYCLE_K, inner=M.INNER_GMRES, t=0.25), M.PCG),
    ("3d-vcycle-cg-inner", (3, 20, 18, 16, 1.0), 0.5, M.DAMPED_JACOBI,
     M.CycleConfig(kind=M.CYCLE_V, inner=M.INNER_CG), M.FGMRES),
    ("2d-sgs", (2, 80, 80, 1, 1.0), 0.25, M.SGS, M.CycleConfig(), M.FGMRES),
    # large coarsest operators: the substitution kernel's multi-row-per-thread paths
    ("2d-two-level-big-coarsest", (2, 150, 150, 1, 1.0), 0.25, M.DAMPED_JACOBI,
     M.CycleConfig(), M.PCG, {"max_levels": 2}),
    ("2d-one-level-4900", (2, 70, 70, 1, 1e-2), 0.25, M.DAMPED_JACOBI, M.CycleConfig(), M.FGMRES,
     {"max_levels": 1}),
]


@pytest.mark.parametrize("case", EXACT_CASES, ids=[c[0] for c in EXACT_CASES])
def test_exact_reduction_mode_bit_identical(gpu, ref, case):
    """aggmg_set_exact_reductions(1) before setup: the reference's 8192-chunk reduction order
    everywhere and the reference's LU substitution on the coarsest level.  The whole solve is
    then bit-identical to the reference: every residual-history entry and the solution."""
    name, (dims, nx, ny, nz, eps), alpha, smoother, cyc, method = case[:6]
    extra = case[6] if len(case) > 6 else {}
    lib = gpu.lib
    lib.fn("set_exact_reductions")(1)
    try:
        A = ref.generate_poisson(dims, nx, ny, nz, eps)
        cfg = M.SetupConfig(alpha=alpha, reuse_caches=True, smoother=smoother, **extra)
        hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
        sc = M.SolverConfig(method=method, tol=1e-8, max_iters=300, restart=30)
        b = np.ones(A.n_rows)
        f, g = (gpu.pcg, ref.pcg) if method == M.PCG else (gpu.fgmres, ref.fgmres)
        rg, rr = f(A, b, None, hg, cyc, sc), g(A, b, None, hr, cyc, sc)
        assert rg.report.iterations == rr.report.iterations
        np.testing.assert_array_equal(bits(np.array(rg.report.residual_history)),
                                      bits(np.array(rr.report.residual_history)))
        np.testing.assert_array_equal(bits(rg.x), bits(rr.x))
    finally:
        lib.fn("set_exact_reductions")(0)


def test_coarsest_zero_pivot(gpu, ref):
    # singular coarsest operator (Neumann 1-D Laplacian, one level): the device Gauss-Jordan
    # reports the reference LU's zero pivot (dense.cpp:42)
    n = 40
    rows, cols, vals = [], [], []
    for i in range(n):
        d = 1.0 if i in (0, n - 1) else 2.0
        rows.append(i); cols.append(i); vals.append(d)
        if i > 0:
            rows.append(i); cols.append(i - 1); vals.append(-1.0)
        if i + 1 < n:
            rows.append(i); cols.append(i + 1); vals.append(-1.0)
    from helpers import from_triplets
    A = from_triplets(n, n, rows, cols, vals)
    cfg = M.SetupConfig(coarse_size_max=100, reuse_caches=True)
    for impl in (gpu, ref):
        with pytest.raises(M.Error, match=f"zero pivot at index {n - 1}"):
            impl.setup_hierarchy(A, None, cfg)


def test_coarsest_inverse_sizes(gpu, ref):
    # one-level hierarchies: the preconditioner is the coarsest direct solve alone
    rng = np.random.default_rng(9)
    for n in (1, 7, 300, 1200):
        A = random_spd(n, min(1.0, 8.0 / n), n)
        cfg = M.SetupConfig(coarse_size_max=2000, reuse_caches=True)
        hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
        r = rng.uniform(-1, 1, n)
        cc = M.CycleConfig(kind=M.CYCLE_V)
        zg, zr = gpu.apply_preconditioner(hg, cc, r), ref.apply_preconditioner(hr, cc, r)
        assert rel_norm(zg, zr) <= 1e-12
