"""CPU: pin the C restatement (oracle/) against the golden fixtures and against the
unmodified reference compiled from /root/reference (oracle/_ref), and re-run the
reference's own known-answer tests on it.  Bit-exact everywhere: the restatement keeps
the reference's evaluation order and is built without FMA."""
import os

import numpy as np
import pytest

from paper_1403_1649_b200 import _abi
from paper_1403_1649_b200 import aggmg as M

import golden_util as G
from helpers import (assert_csr_bits, assert_pattern, bits, laplacian_1d, random_graph,
                     random_sparse, random_spd)

from oracle.checkers import REF_LIB  # noqa: E402

HAVE_REF = os.path.exists(REF_LIB)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="reference shim not built")


@pytest.mark.parametrize("name", G.HIERARCHY_CASES)
def test_oracle_matches_golden_hierarchy(orc, name):
    G.check_hierarchy(orc, name, exact_solve=True)


def test_oracle_worked_example_golden(orc):
    d = G.load("worked_example")
    A = G.csr(d, "A")
    agg = M.Aggregation(8, 3, d["assignment"], np.array([1, 0, 2]))
    c = orc.build_galerkin_cache(A, agg)
    for f in ("entry", "entry_row", "segment_offsets", "slot_of_csr"):
        np.testing.assert_array_equal(getattr(c, f), d[f])
    P = M.SparseMatrix(8, 3, np.arange(9), d["assignment"], np.ones(8))
    assert_csr_bits(orc.apply_galerkin_cache(c, A, P), G.csr(d, "Ac"))


def test_oracle_mis2_golden(orc):
    d = G.load("mis2_grid")
    S = G.csr(d, "S")
    for key in [k for k in d if k.startswith("state_")]:
        seed = int(key[len("state_"):])
        np.testing.assert_array_equal(orc.mis2(S, d["influence"], seed).state, d[key])


# ---- the reference's own known-answer tests, re-run on the restatement ---------------


def test_worked_example_exact_sums(orc):
    """test_galerkin.cpp:70-92: seven coarse pairs, power-of-two sums exact."""
    d = G.load("worked_example")
    A = G.csr(d, "A")
    a = d["assignment"]
    P = M.SparseMatrix(8, 3, np.arange(9), a, np.ones(8))
    R = orc.transpose(P)
    Ac = orc.galerkin_direct(R, A, P)
    assert list(Ac.row_offsets) == [0, 3, 5, 7]
    assert list(Ac.col_indices) == [0, 1, 2, 0, 1, 0, 2]
    at = lambda i, j: A.at(i - 1, j - 1)  # noqa: E731  (1-based names as in the paper)
    assert Ac.at(0, 0) == sum(at(i, j) for i in (2, 4, 7) for j in (2, 4, 7))
    assert Ac.at(0, 1) == at(2, 1) + at(4, 6)
    assert Ac.at(0, 2) == at(4, 5)
    assert Ac.at(1, 0) == at(1, 2) + at(6, 4)
    assert Ac.at(1, 1) == at(1, 1) + at(1, 6) + at(6, 1) + at(6, 6)
    assert Ac.at(2, 0) == at(5, 4)
    assert Ac.at(2, 2) == sum(at(i, j) for i in (3, 5, 8) for j in (3, 5, 8))


def test_strength_hand_cases(orc):
    """test_strength.cpp:25-112: ties at the threshold are weak, the row max is strong,
    sign follows the diagonal."""
    A = M.SparseMatrix(3, 3, np.array([0, 3, 5, 7]), np.array([0, 1, 2, 0, 1, 1, 2]),
                       np.array([4.0, -2.0, -0.5, -1.0, 3.0, -1.0, 2.0]))
    C = orc.classic_strength(A, 0.25)
    assert list(C.row_offsets) == [0, 1, 2, 3] and list(C.col_indices) == [1, 0, 1]
    T = M.SparseMatrix(1, 3, np.array([0, 3]), np.array([0, 1, 2]), np.array([1.0, -1.0, -0.25]))
    T = M.SparseMatrix(3, 3, np.array([0, 3, 3, 3]), T.col_indices, T.values)
    C = orc.classic_strength(T, 0.25)
    assert list(C.col_indices) == [1]  # -0.25 == 0.25 * 1.0 exactly: weak
    N = M.SparseMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]),
                       np.array([-2.0, 1.0, 1.0, -2.0]))
    assert list(orc.classic_strength(N, 0.5).col_indices) == [1, 0]  # negative diagonal


def test_mis2_small_graphs(orc):
    """test_aggregation.cpp:67-105: isolated nodes are roots; a path roots the middle;
    a star roots the hub."""
    iso = M.SparseMatrix(5, 5, np.zeros(6, dtype=np.int64), np.array([], dtype=np.int64),
                         np.array([]))
    assert np.all(orc.mis2(iso, np.zeros(5, dtype=np.int64), 1).state == 1)
    path = random_graph(3, 0.0, 0)
    path = M.SparseMatrix(3, 3, np.array([0, 1, 3, 4]), np.array([1, 0, 2, 1]), np.ones(4))
    st = orc.mis2(path, np.array([1, 2, 1]), 5).state
    assert list(st) == [-1, 1, -1]
    n = 9
    rows = [0] * (n - 1) + list(range(1, n))
    cols = list(range(1, n)) + [0] * (n - 1)
    from helpers import from_triplets
    star = from_triplets(n, n, rows, cols, np.ones(2 * (n - 1)))
    st = orc.mis2(star, np.array([n - 1] + [1] * (n - 1)), 3).state
    assert st[0] == 1 and np.all(st[1:] == -1)


def bfs_ok(S, state):
    """Independence at distance 2 and maximality, by BFS (test_helpers.hpp:224-243)."""
    roots = np.nonzero(state == 1)[0]
    n = S.n_rows
    dist = np.full(n, 99)
    for r in roots:
        d = {r: 0}
        frontier = [r]
        for step in (1, 2):
            nxt = []
            for u in frontier:
                for v in S.col_indices[S.row_offsets[u]:S.row_offsets[u + 1]]:
                    if v not in d:
                        d[v] = step
                        nxt.append(v)
            frontier = nxt
        for v, dv in d.items():
            if v != r and state[v] == 1:
                return False
            dist[v] = min(dist[v], dv)
    return bool(np.all(dist <= 2))


def test_mis2_bfs_properties(orc):
    """test_aggregation.cpp:107-122 / acceptance criterion 6 on seeded random graphs."""
    for seed in range(40):
        S = random_graph(30 + seed % 20, 0.08, 900 + seed)
        infl = orc.influence_counts(S)
        assert bfs_ok(S, orc.mis2(S, infl, seed).state), seed


def test_pass2_tie_break(orc):
    """test_aggregation.cpp:178-204: pass 2 takes the heaviest |A| edge, ties to the
    lower aggregate id."""
    # 0 - 1 - 2 - 3 - 4 path; roots 0 and 4 -> 1 and 3 join in pass 1; 2 decides in pass 2
    S = M.SparseMatrix(5, 5, np.array([0, 1, 3, 5, 7, 8]), np.array([1, 0, 2, 1, 3, 2, 4, 3]),
                       np.ones(8))
    state = np.array([1, -1, -1, -1, 1], dtype=np.int8)
    for w12, w23, want in ((-1.0, -1.0, 0), (-1.0, -2.0, 1), (-3.0, -2.0, 0)):
        A = M.SparseMatrix(5, 5, np.array([0, 2, 5, 8, 11, 13]),
                           np.array([0, 1, 0, 1, 2, 1, 2, 3, 2, 3, 4, 3, 4]),
                           np.array([2, -1, -1, 2, w12, w12, 2, w23, w23, 2, -1, -1, 2.0]))
        agg = orc.aggregate(S, A, M.Mis2Result(state, np.array([0, 4]), 1))
        assert agg.assignment[2] == want, (w12, w23)


def test_transfer_hand_case(orc):
    """test_transfer.cpp:21-34: P = [[1/sqrt2,0],[1/sqrt2,0],[0,1]]."""
    agg = M.Aggregation(3, 2, np.array([0, 0, 1]), np.array([0, 2]))
    t = orc.build_transfer(agg, np.ones(3))
    assert np.allclose(t.P.to_dense(), [[2 ** -0.5, 0], [2 ** -0.5, 0], [0, 1]], atol=0, rtol=1e-15)
    assert np.array_equal(t.coarse_b, [np.sqrt(2.0), 1.0])


def test_omega_diagonal_exact(orc):
    """test_smoother.cpp:40-54 / acceptance criterion 7: diagonal matrices give 4/3."""
    D = M.SparseMatrix(4, 4, np.arange(5), np.arange(4), np.array([2.0, 4.0, 0.5, 8.0]))
    assert orc.setup_smoother(D, M.DAMPED_JACOBI, 5, 3).omega == 4.0 / 3.0
    s = orc.setup_smoother(laplacian_1d(200), M.DAMPED_JACOBI, 5, 1)
    assert abs(s.omega - 2.0 / 3.0) <= 0.05 * 2.0 / 3.0


# ---- restatement vs the reference itself ----------------------------------------------


@needs_ref
def test_components_match_reference(orc, ref):
    rng = np.random.default_rng(0)
    for seed in range(8):
        A = random_sparse(80 + seed, 80 + seed, 0.07, seed)
        assert_pattern(orc.classic_strength(A, 0.3), ref.classic_strength(A, 0.3))
        Cm = ref.classic_strength(A, 0.3)
        np.testing.assert_array_equal(orc.influence_counts(Cm), ref.influence_counts(Cm))
        S = ref.symmetrize_pattern(Cm)
        assert_pattern(orc.symmetrize_pattern(Cm), S)
        infl = ref.influence_counts(Cm)
        mo, mr = orc.mis2(S, infl, seed), ref.mis2(S, infl, seed)
        np.testing.assert_array_equal(mo.state, mr.state)
        assert mo.sweeps == mr.sweeps
        ao, ar = orc.aggregate(S, A, mr), ref.aggregate(S, A, mr)
        np.testing.assert_array_equal(ao.assignment, ar.assignment)
        np.testing.assert_array_equal(ao.representatives, ar.representatives)
        b = rng.uniform(0.5, 2.0, A.n_rows)
        to, tr = orc.build_transfer(ar, b), ref.build_transfer(ar, b)
        assert_csr_bits(to.P, tr.P)
        assert_csr_bits(to.R, tr.R)
        co, cr = orc.build_galerkin_cache(A, ar), ref.build_galerkin_cache(A, ar)
        for f in ("entry", "entry_row", "segment_offsets", "slot_of_csr", "rows_by_coarse"):
            np.testing.assert_array_equal(getattr(co, f), getattr(cr, f))
        assert_csr_bits(orc.apply_galerkin_cache(co, A, tr.P), ref.apply_galerkin_cache(cr, A, tr.P))
        assert_csr_bits(orc.galerkin_direct(tr.R, A, tr.P), ref.galerkin_direct(tr.R, A, tr.P))
        x = rng.uniform(-1, 1, A.n_rows)
        np.testing.assert_array_equal(bits(orc.spmv(A, x)), bits(ref.spmv(A, x)))


@needs_ref
def test_smoother_and_eigs_match_reference(orc, ref):
    for seed in range(5):
        A = random_spd(60 + 10 * seed, 0.1, seed)
        so, sr = orc.setup_smoother(A, M.DAMPED_JACOBI, 5, seed), ref.setup_smoother(A, M.DAMPED_JACOBI, 5, seed)
        assert so.omega == sr.omega and so.rho_est == sr.rho_est
        b, x = np.ones(A.n_rows), np.linspace(-1, 1, A.n_rows)
        for kind in (M.JACOBI, M.DAMPED_JACOBI, M.SGS):
            st = M.SmootherState(kind, sr.inv_diag, sr.omega, sr.rho_est)
            np.testing.assert_array_equal(bits(orc.smooth(st, A, b, x)), bits(ref.smooth(st, A, b, x)))
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 4, 5):
        H = np.triu(rng.uniform(-1, 1, (n, n)), -1)
        eo, er = orc.hessenberg_eigenvalues(H), ref.hessenberg_eigenvalues(H)
        np.testing.assert_array_equal(bits(eo.real), bits(er.real))
        np.testing.assert_array_equal(bits(eo.imag), bits(er.imag))


@needs_ref
@pytest.mark.parametrize("reuse", [True, False])
def test_solves_match_reference_bitwise(orc, ref, reuse):
    for A, alpha in ((ref.generate_poisson(2, 48, 40, 1, 0.01), 0.25),
                     (ref.generate_poisson(3, 16, 16, 16), 0.5)):
        cfg = M.SetupConfig(alpha=alpha, coarse_size_max=40, reuse_caches=reuse)
        ho, hr = orc.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
        for f, restart in (("pcg", 30), ("fgmres", 6)):
            for cc in (M.CycleConfig(), M.CycleConfig(kind=M.CYCLE_V),
                       M.CycleConfig(kind=M.CYCLE_K, inner=M.INNER_CG)):
                sc = M.SolverConfig(method=M.PCG if f == "pcg" else M.FGMRES, tol=1e-9,
                                    max_iters=200, restart=restart)
                ro = getattr(orc, f)(A, np.ones(A.n_rows), None, ho, cc, sc)
                rr = getattr(ref, f)(A, np.ones(A.n_rows), None, hr, cc, sc)
                np.testing.assert_array_equal(bits(ro.report.residual_history),
                                              bits(rr.report.residual_history))
                np.testing.assert_array_equal(bits(ro.x), bits(rr.x))


@needs_ref
def test_refresh_matches_reference(orc, ref):
    A = ref.generate_poisson(2, 30, 30)
    cfg = M.SetupConfig(reuse_caches=True, coarse_size_max=30)
    ho, hr = orc.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    v = A.values * 1.5
    orc.refresh_values(ho, v)
    ref.refresh_values(hr, v)
    for lo, lr in zip(ho.levels, hr.levels):
        assert_csr_bits(lo.A, lr.A)
    h0 = orc.setup_hierarchy(A, None, M.SetupConfig(coarse_size_max=30))
    with pytest.raises(M.Error, match="without caches"):
        orc.refresh_values(h0, v)


def test_errors_match_reference_messages(orc):
    with pytest.raises(M.Error, match="too large"):
        orc.setup_hierarchy(orc.generate_poisson(2, 80, 80), None,
                            M.SetupConfig(max_levels=1, coarse_size_max=10))
    bad = M.SparseMatrix(2, 2, np.array([0, 2, 3]), np.array([1, 0, 1]), np.ones(3))
    with pytest.raises(M.Error, match="strictly increasing in row 0"):
        orc.setup_hierarchy(bad)
    A = M.SparseMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, -1.0]))
    with pytest.raises(M.Error, match="use fgmres"):
        orc.pcg(A, np.ones(2), None, None, None, M.SolverConfig(method=M.PCG))
