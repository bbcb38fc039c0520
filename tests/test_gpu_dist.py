"""Row-partitioned (multi-GPU) path, run as R rank threads on one B200 (in-process transport;
the NCCL transport carries the same bytes between processes).

Bar: for every rank count, aggregates / P / B / coarse operators are bit-identical
to the one-GPU hierarchy (which is itself bit-identical to the reference cache path), omega
within 1e-12, and the partitioned PCG / FGMRES reach the one-GPU iteration counts with
residual histories within 1e-10 * ||r0|| (one rank: bit-identical)."""
import threading

import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M
from paper_1403_1649_b200 import dist as D

from helpers import bits, random_spd

pytestmark = pytest.mark.gpu


def problems(gpu):
    yield "2d-64x40", gpu.generate_poisson(2, 64, 40), 0.25
    yield "3d-18", gpu.generate_poisson(3, 18, 18, 18), 0.5
    yield "3d-aniso-20x16x12", gpu.generate_poisson(3, 20, 16, 12, 1e-3), 0.5
    yield "jump27-12", gpu.generate_jump27(12, 12, 12, 1e6, 3), 0.5
    yield "spd-500", random_spd(500, 0.02, 21), 0.25


def run_dist(A, P, cfg, agglomerate, solver=None, cycle=None, part=None):
    """Setup (+ optional solve) on P rank threads; rank 0's gathered results."""
    out = {}
    lock = threading.Lock()

    def rank_fn(comm, r):
        dA = D.DistMatrix.from_global(comm, A, part)
        h = D.setup(comm, dA, cfg, agglomerate_rows=agglomerate)
        res = {"info": h.info(), "levels": []}
        nl = h.n_levels()
        for k in range(nl):
            Ak = h.level_A(k)
            tr = h.level_transfer(k) if k + 1 < nl else None
            Bk = h.level_B(k)
            om = h.level_omega(k)
            res["levels"].append((Ak, tr, Bk, om))
        res["warnings"] = h.warnings()
        if solver is not None:
            n0, row0, nloc, _ = dA.info()
            res["solve"] = h.solve(solver, cycle, n_local=nloc)
            res["row0"] = row0
        h.free()
        dA.free()
        with lock:
            out[r] = res

    D.run_threads(P, rank_fn)
    return out


def compare_hierarchy(hg, res, name):
    lv = res[0]["levels"]
    assert len(lv) == hg.n_levels(), f"{name}: level count {len(lv)} vs {hg.n_levels()}"
    for k, (Ak, tr, Bk, om) in enumerate(lv):
        L = hg.levels[k]
        Ag = L.A
        assert np.array_equal(Ak.row_offsets, Ag.row_offsets), f"{name} L{k} rowptr"
        assert np.array_equal(Ak.col_indices, Ag.col_indices), f"{name} L{k} cols"
        assert np.array_equal(bits(Ak.values), bits(Ag.values)), f"{name} L{k} values"
        assert np.array_equal(bits(Bk), bits(L.B)), f"{name} L{k} B"
        if tr is not None:
            a, p, sweeps = tr
            ag, ncg, swg = L.aggregation()
            assert np.array_equal(a, ag), f"{name} L{k} aggregates"
            assert sweeps == swg, f"{name} L{k} MIS sweeps {sweeps} vs {swg}"
            Pg = L.P
            nz = p != 0.0
            assert np.array_equal(bits(p[nz]), bits(Pg.values)), f"{name} L{k} P values"
            omg = L.smoother.omega
            assert abs(om - omg) <= 1e-12 * abs(omg), f"{name} L{k} omega {om} vs {omg}"


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_dist_setup_bit_exact(gpu, P):
    for name, A, alpha in problems(gpu):
        cfg = M.SetupConfig(alpha=alpha, reuse_caches=True, coarse_size_max=40)
        hg = gpu.setup_hierarchy(A, None, cfg)
        res = run_dist(A, P, cfg, agglomerate=60)
        assert res[0]["info"][1] >= 1, f"{name}: nothing distributed"
        compare_hierarchy(hg, res, f"{name} P={P}")


def test_dist_uneven_partition(gpu):
    A = gpu.generate_poisson(3, 16, 14, 12)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=30)
    hg = gpu.setup_hierarchy(A, None, cfg)
    n = A.n_rows
    part = [0, 7, n // 3, n // 3 + 1, n]  # a 1-row rank and a 7-row rank
    res = run_dist(A, 4, cfg, agglomerate=50, part=part)
    compare_hierarchy(hg, res, "uneven")


@pytest.mark.parametrize("method", ["pcg", "fgmres"])
@pytest.mark.parametrize("P", [1, 2, 4])
def test_dist_solve_matches_one_gpu(gpu, P, method):
    A = gpu.generate_poisson(3, 24, 22, 20)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=60)
    sc = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=1e-8, max_iters=200,
                        restart=30)
    cyc = M.CycleConfig()
    hg = gpu.setup_hierarchy(A, None, cfg)
    b = np.ones(A.n_rows)
    rg = gpu.pcg(A, b, None, hg, cyc, sc) if method == "pcg" else gpu.fgmres(A, b, None, hg, cyc, sc)
    res = run_dist(A, P, cfg, agglomerate=400, solver=sc, cycle=cyc)
    s0 = res[0]["solve"]
    assert s0.report.converged
    assert s0.report.iterations == rg.report.iterations
    hd, hs = np.array(s0.report.residual_history), np.array(rg.report.residual_history)
    if P == 1:
        assert np.array_equal(bits(hd), bits(hs)), "one rank must be bit-identical"
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0]
    x = np.zeros(A.n_rows)
    for r, rr in res.items():
        sl = rr["solve"].x
        x[rr["row0"]:rr["row0"] + sl.shape[0]] = sl
    assert np.max(np.abs(x - rg.x)) <= 1e-10 * np.max(np.abs(rg.x))


def test_dist_generated_matches_host_slices(gpu):
    """Device slab generators == slices of the one-GPU generator (same global matrix)."""
    out = {}

    def rank_fn(comm, r):
        dA = D.DistMatrix.poisson(comm, 3, 10, 9, 8)
        h = D.setup(comm, dA, M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=20),
                    agglomerate_rows=30)
        out[r] = h.level_A(0)
        h.free()
        dA.free()

    D.run_threads(3, rank_fn)
    A = gpu.generate_poisson(3, 10, 9, 8)
    assert np.array_equal(out[0].col_indices, A.col_indices)
    assert np.array_equal(bits(out[0].values), bits(A.values))


def test_dist_errors_propagate(gpu):
    # structurally non-symmetric operator: the partitioned strength graph leaves the halo
    n = 40
    rows, cols, vals = [], [], []
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(4.0)
        if i + 1 < n:
            rows.append(i); cols.append(i + 1); vals.append(-1.0)
        if i >= 21:
            rows.append(i); cols.append(i - 21); vals.append(-1.5)
    from helpers import from_triplets
    A = from_triplets(n, n, rows, cols, vals)
    cfg = M.SetupConfig(alpha=0.25, reuse_caches=True, coarse_size_max=4)
    with pytest.raises(M.Error, match="structurally symmetric|rank"):
        run_dist(A, 2, cfg, agglomerate=5)


def test_dist_rejects_sgs(gpu):
    # sgs is one global sequential sweep: a row partition cannot reproduce it
    A = gpu.generate_poisson(2, 16, 16)
    cfg = M.SetupConfig(alpha=0.25, reuse_caches=True, coarse_size_max=10, smoother=M.SGS)
    with pytest.raises(M.Error, match="sgs"):
        run_dist(A, 2, cfg, agglomerate=50)


def test_dist_aniso_fgmres_three_ranks_uneven(gpu):
    A = gpu.generate_poisson(3, 22, 18, 16, 1e-3)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=50)
    sc = M.SolverConfig(method=M.FGMRES, tol=1e-8, max_iters=300, restart=30)
    hg = gpu.setup_hierarchy(A, None, cfg)
    rg = gpu.fgmres(A, np.ones(A.n_rows), None, hg, M.CycleConfig(), sc)
    n = A.n_rows
    part = [0, n // 5, n // 2 + 17, n]
    res = run_dist(A, 3, cfg, agglomerate=300, solver=sc, cycle=M.CycleConfig(), part=part)
    compare_hierarchy(hg, res, "aniso P=3")
    s0 = res[0]["solve"]
    assert s0.report.iterations == rg.report.iterations
    hd, hs = np.array(s0.report.residual_history), np.array(rg.report.residual_history)
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0]


def test_dist_jump27_pcg_two_ranks(gpu):
    A = gpu.generate_jump27(14, 13, 12, 1e6, 4)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=40)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=300)
    hg = gpu.setup_hierarchy(A, None, cfg)
    rg = gpu.pcg(A, np.ones(A.n_rows), None, hg, M.CycleConfig(), sc)
    res = run_dist(A, 2, cfg, agglomerate=150, solver=sc, cycle=M.CycleConfig())
    compare_hierarchy(hg, res, "jump27 P=2")
    s0 = res[0]["solve"]
    assert s0.report.iterations == rg.report.iterations
    hd, hs = np.array(s0.report.residual_history), np.array(rg.report.residual_history)
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0]


@pytest.mark.parametrize("P", [1, 2])
def test_dist_preconditioner_matches_one_gpu(gpu, P):
    A = gpu.generate_poisson(3, 20, 20, 20)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=40)
    hg = gpu.setup_hierarchy(A, None, cfg)
    r = np.random.default_rng(9).uniform(-1, 1, A.n_rows)
    zg = gpu.apply_preconditioner(hg, M.CycleConfig(), r)
    n = A.n_rows
    out = {}

    def fn(comm, k):
        dA = D.DistMatrix.from_global(comm, A)
        h = D.setup(comm, dA, cfg, agglomerate_rows=100)
        _, row0, nloc, _ = dA.info()
        out[k] = (row0, h.apply_preconditioner(r[row0:row0 + nloc]))
        h.free()
        dA.free()

    D.run_threads(P, fn)
    z = np.zeros(n)
    for row0, zl in out.values():
        z[row0:row0 + zl.shape[0]] = zl
    if P == 1:
        assert np.array_equal(z.view(np.uint64), zg.view(np.uint64))
    else:
        assert np.max(np.abs(z - zg)) <= 1e-12 * np.max(np.abs(zg))


@pytest.mark.parametrize("P", [1, 3])
def test_dist_refresh_values_matches_one_gpu(gpu, P):
    """refresh_values on the ranks == refresh_values on one GPU (hierarchy.cpp:90-104)."""
    A = gpu.generate_poisson(3, 18, 17, 16, 0.3)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True, coarse_size_max=40)
    rng = np.random.default_rng(4)
    newv = A.values * rng.uniform(0.5, 1.5, A.values.shape[0])  # same pattern, new values
    Anew = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, newv)
    hg = gpu.setup_hierarchy(A, None, cfg)
    hg = gpu.refresh_values(hg, newv)
    out = {}

    def fn(comm, r):
        dA = D.DistMatrix.from_global(comm, A)
        h = D.setup(comm, dA, cfg, agglomerate_rows=120)
        _, row0, nloc, _ = dA.info()
        lo, hi = A.row_offsets[row0], A.row_offsets[row0 + nloc]
        h.refresh_values(newv[lo:hi])
        res = {"levels": []}
        for k in range(h.n_levels()):
            res["levels"].append((h.level_A(k), h.level_transfer(k) if k + 1 < h.n_levels() else None,
                                  h.level_B(k), h.level_omega(k)))
        out[r] = res
        h.free()
        dA.free()

    D.run_threads(P, fn)
    compare_hierarchy(hg, out, f"refresh P={P}")
    del Anew


@pytest.mark.parametrize("P", [1, 2])
def test_dist_sell_operators_match_one_gpu(gpu, P):
    # local slabs past the SELL-32 threshold (>= 2^19 rows per rank): the partitioned sweeps run
    # SELL over the interior / boundary row sub-ranges; same iterations, histories within 1e-10,
    # one rank bit-identical
    A = gpu.generate_poisson(3, 104, 104, 104)
    assert A.n_rows // P >= 1 << 19
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    cyc = M.CycleConfig()
    hg = gpu.setup_hierarchy(A, None, cfg)
    rg = gpu.pcg(A, np.ones(A.n_rows), None, hg, cyc, sc)
    res = run_dist(A, P, cfg, agglomerate=100_000, solver=sc, cycle=cyc)
    assert res[0]["info"][1] >= 1  # at least level 0 partitioned
    s0 = res[0]["solve"]
    assert s0.report.iterations == rg.report.iterations
    hd, hs = np.array(s0.report.residual_history), np.array(rg.report.residual_history)
    if P == 1:
        assert np.array_equal(bits(hd), bits(hs))
    assert np.max(np.abs(hd - hs)) <= 1e-10 * hs[0]
