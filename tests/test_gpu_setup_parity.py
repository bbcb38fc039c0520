"""Setup-stage parity: every B200 setup kernel against the unmodified reference
(oracle/_ref) on the same inputs.  Bar: bit-exact patterns, aggregates,
P/R/B and coarse values (cache summation order); omega within 1e-12."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import (assert_csr_bits, assert_pattern, bits, laplacian_1d, random_graph,
                     random_sparse, random_spd)

pytestmark = pytest.mark.gpu


def problems(ref):
    yield "2d-48", ref.generate_poisson(2, 48, 48), 0.25
    yield "2d-aniso-40x33", ref.generate_poisson(2, 40, 33, 1, 0.01), 0.25
    yield "3d-14", ref.generate_poisson(3, 14, 14, 14), 0.5
    yield "3d-aniso-16x12x10", ref.generate_poisson(3, 16, 12, 10, 1e-3), 0.5
    yield "jump27-10", M.b200().generate_jump27(10, 10, 10, 1e6, 3), 0.5
    yield "spd-300", random_spd(300, 0.03, 11), 0.25
    yield "lap1d-257", laplacian_1d(257), 0.25


def each_problem(ref):
    for name, A, alpha in problems(ref):
        if A is not None:
            yield name, A, alpha


def test_strength_bit_exact(gpu, ref):
    for name, A, alpha in each_problem(ref):
        for a in (alpha, 0.5, 0.9):
            assert_pattern(gpu.classic_strength(A, a), ref.classic_strength(A, a), f"{name} a={a}")
    A = random_sparse(120, 120, 0.08, 5)  # mixed signs, zero / missing diagonals
    assert_pattern(gpu.classic_strength(A, 0.3), ref.classic_strength(A, 0.3), "random")


def test_strength_errors(gpu, ref):
    A = random_sparse(40, 40, 0.1, 1)
    with pytest.raises(M.Error, match="alpha"):
        gpu.classic_strength(A, 1.5)
    D = laplacian_1d(10)
    D.values[D.row_offsets[3] + 1] = 0.0  # zero diagonal at row 3
    with pytest.raises(M.Error, match="diagonal at row 3"):
        gpu.classic_strength(D, 0.25, M.ZERO_DIAG_FAIL)


def test_influence_and_symmetrize(gpu, ref):
    for seed in range(6):
        A = random_sparse(150, 150, 0.05, 100 + seed)
        Cm = ref.classic_strength(A, 0.25)
        np.testing.assert_array_equal(gpu.influence_counts(Cm), ref.influence_counts(Cm))
        assert_pattern(gpu.symmetrize_pattern(Cm), ref.symmetrize_pattern(Cm), f"seed {seed}")


def test_mis2_bit_exact(gpu, ref):
    cases = [random_graph(200, 0.03, s) for s in range(5)]
    cases += [random_graph(60, 0.0, 1)]  # isolated nodes
    for name, A, alpha in each_problem(ref):
        cases.append(ref.symmetrize_pattern(ref.classic_strength(A, alpha)))
    for i, S in enumerate(cases):
        infl = ref.influence_counts(S)
        for seed in (0, 42, 2**63 + 5):
            g, r = gpu.mis2(S, infl, seed), ref.mis2(S, infl, seed)
            np.testing.assert_array_equal(g.state, r.state, err_msg=f"case {i} seed {seed}")
            assert g.sweeps == r.sweeps, (i, seed)


def test_aggregate_bit_exact(gpu, ref):
    for name, A, alpha in each_problem(ref):
        S = ref.symmetrize_pattern(ref.classic_strength(A, alpha))
        mis = ref.mis2(S, ref.influence_counts(ref.classic_strength(A, alpha)), 7)
        g, r = gpu.aggregate(S, A, mis), ref.aggregate(S, A, mis)
        assert g.n_aggregates == r.n_aggregates, name
        np.testing.assert_array_equal(g.assignment, r.assignment, err_msg=name)
        np.testing.assert_array_equal(g.representatives, r.representatives, err_msg=name)


def test_transfer_bit_exact(gpu, ref):
    rng = np.random.default_rng(3)
    for n, nc in ((50, 7), (400, 33), (1000, 1)):
        a = np.concatenate([np.arange(nc), rng.integers(0, nc, n - nc)]).astype(np.int64)
        agg = M.Aggregation(n, nc, a, np.zeros(nc, dtype=np.int64))
        for b in (np.ones(n), rng.uniform(-1, 1, n), np.where(np.arange(n) % 5 == 0, 0.0, 1.5)):
            if any(np.all(b[a == J] == 0) for J in range(nc)):
                continue
            tg, tr = gpu.build_transfer(agg, b), ref.build_transfer(agg, b)
            assert_csr_bits(tg.P, tr.P, "P")
            assert_csr_bits(tg.R, tr.R, "R")
            np.testing.assert_array_equal(bits(tg.coarse_b), bits(tr.coarse_b))
    agg = M.Aggregation(4, 2, np.array([0, 0, 1, 1]), np.array([0, 2]))
    with pytest.raises(M.Error, match="aggregate 1"):
        gpu.build_transfer(agg, np.array([1.0, 2.0, 0.0, 0.0]))


def test_galerkin_cache_bit_exact(gpu, ref):
    rng = np.random.default_rng(9)
    for seed in range(4):
        n = 60 + 17 * seed
        nc = 3 + seed * 5
        A = random_sparse(n, n, 0.15, 7000 + seed)
        a = np.concatenate([np.arange(nc), rng.integers(0, nc, n - nc)]).astype(np.int64)
        agg = M.Aggregation(n, nc, a, np.zeros(nc, dtype=np.int64))
        cg, cr = gpu.build_galerkin_cache(A, agg), ref.build_galerkin_cache(A, agg)
        for f in ("coarse_row_offsets", "coarse_col_indices", "entry", "entry_row",
                  "segment_offsets", "slot_of_csr", "rows_by_coarse", "agg_row_offsets"):
            np.testing.assert_array_equal(getattr(cg, f), getattr(cr, f), err_msg=f)
        P = ref.build_transfer(agg, rng.uniform(0.5, 1.5, n)).P
        assert_csr_bits(gpu.apply_galerkin_cache(cg, A, P), ref.apply_galerkin_cache(cr, A, P))


def test_galerkin_cache_large_segment_fallback(gpu, ref):
    # one aggregate holding every row: a single coarse row whose segment exceeds the
    # shared-memory path (> 1024 fine entries)
    A = random_spd(700, 0.01, 4)
    agg = M.Aggregation(700, 2, (np.arange(700) % 2).astype(np.int64), np.array([0, 1]))
    cg, cr = gpu.build_galerkin_cache(A, agg), ref.build_galerkin_cache(A, agg)
    np.testing.assert_array_equal(cg.entry, cr.entry)
    np.testing.assert_array_equal(cg.segment_offsets, cr.segment_offsets)
    P = ref.build_transfer(agg, np.ones(700)).P
    assert_csr_bits(gpu.apply_galerkin_cache(cg, A, P), ref.apply_galerkin_cache(cr, A, P))


def test_galerkin_cache_refuses_changed_pattern(gpu, ref):
    A = random_spd(30, 0.2, 2)
    agg = M.Aggregation(30, 3, (np.arange(30) % 3).astype(np.int64), np.arange(3))
    c = gpu.build_galerkin_cache(A, agg)
    P = ref.build_transfer(agg, np.ones(30)).P
    B = random_spd(30, 0.3, 5)
    with pytest.raises(M.Error, match="rebuild"):
        gpu.apply_galerkin_cache(c, B, P)


def test_smoother_setup(gpu, ref):
    for name, A, alpha in each_problem(ref):
        for seed in (0, 12345):
            g = gpu.setup_smoother(A, M.DAMPED_JACOBI, 5, seed)
            r = ref.setup_smoother(A, M.DAMPED_JACOBI, 5, seed)
            np.testing.assert_array_equal(bits(g.inv_diag), bits(r.inv_diag))
            # reference-order Arnoldi dots + the reference's Francis QR: omega bit-identical
            assert g.omega == r.omega and g.rho_est == r.rho_est, (name, g.omega, r.omega)
    D = M.SparseMatrix(4, 4, np.arange(5), np.arange(4), np.array([2.0, 4.0, 0.5, 8.0]))
    s = gpu.setup_smoother(D, M.DAMPED_JACOBI, 5, 3)
    assert s.omega == 4.0 / 3.0  # smoother.cpp:31-36: diagonal matrices give exactly 4/3


@pytest.mark.parametrize("case", ["2d-64", "2d-aniso-80x50", "3d-20", "3d-aniso-24", "spd-500"])
def test_hierarchy_bit_exact(gpu, ref, case):
    A, alpha = {
        "2d-64": (lambda: ref.generate_poisson(2, 64, 64), 0.25),
        "2d-aniso-80x50": (lambda: ref.generate_poisson(2, 80, 50, 1, 0.01), 0.25),
        "3d-20": (lambda: ref.generate_poisson(3, 20, 20, 20), 0.5),
        "3d-aniso-24": (lambda: ref.generate_poisson(3, 24, 24, 24, 1e-3), 0.5),
        "spd-500": (lambda: random_spd(500, 0.02, 77), 0.25),
    }[case]
    A = A()
    cfg = M.SetupConfig(alpha=alpha, coarse_size_max=50, reuse_caches=True)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    assert hg.n_levels() == hr.n_levels()
    assert hg.warnings == hr.warnings
    for k, (lg, lr) in enumerate(zip(hg.levels, hr.levels)):
        assert_csr_bits(lg.A, lr.A, f"A level {k}")
        np.testing.assert_array_equal(bits(lg.B), bits(lr.B), err_msg=f"B level {k}")
        if k < hg.coarsest():
            assert_csr_bits(lg.P, lr.P, f"P level {k}")
            assert_csr_bits(lg.R, lr.R, f"R level {k}")
            sg, sr = lg.smoother, lr.smoother
            np.testing.assert_array_equal(bits(sg.inv_diag), bits(sr.inv_diag))
            assert sg.omega == sr.omega


def test_hierarchy_errors(gpu, ref):
    A = ref.generate_poisson(2, 8, 8)
    with pytest.raises(M.Error, match="zero"):
        gpu.setup_hierarchy(A, np.zeros(64))
    bad = M.SparseMatrix(2, 2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))
    with pytest.raises(M.Error, match="strictly increasing in row 0"):
        gpu.setup_hierarchy(bad)
    big = ref.generate_poisson(2, 80, 80)
    with pytest.raises(M.Error, match="too large"):
        gpu.setup_hierarchy(big, None, M.SetupConfig(max_levels=1, coarse_size_max=10))


def test_stall_warning(gpu, ref):
    D = M.SparseMatrix(700, 700, np.arange(701), np.arange(700), np.full(700, 3.0))
    hg = gpu.setup_hierarchy(D)
    hr = ref.setup_hierarchy(D)
    assert hg.warnings == hr.warnings and "stalled" in hg.warnings[0]


def test_hessenberg_eigenvalues_bit_exact(gpu, ref):
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 4, 5):
        for _ in range(5):
            H = np.triu(rng.uniform(-1, 1, (n, n)), -1)
            eg, er = gpu.hessenberg_eigenvalues(H), ref.hessenberg_eigenvalues(H)
            np.testing.assert_array_equal(bits(eg.real), bits(er.real))
            np.testing.assert_array_equal(bits(eg.imag), bits(er.imag))
