"""Load the golden fixtures (tests/golden/*.npz, produced from the unmodified reference
by tests/golden/make_golden.py) and check any backend against them."""
import os

import numpy as np

from paper_1403_1649_b200 import aggmg as M

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
HIERARCHY_CASES = ["poisson2d_32", "aniso2d_40x24", "poisson3d_12", "aniso3d_14"]


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def csr(d, prefix):
    n, m = d[f"{prefix}_shape"]
    return M.SparseMatrix(int(n), int(m), d[f"{prefix}_ro"], d[f"{prefix}_ci"], d[f"{prefix}_v"])


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def check_hierarchy(backend, name, exact_solve=True):
    """Setup must be bit-identical to the reference; the solve too when exact_solve,
    else iteration count equal and history within 1e-10 of the initial residual."""
    d = load(name)
    dims, nx, ny, nz = (int(v) for v in d["spec"])
    A = backend.generate_poisson(dims, nx, ny, nz, float(d["epsilon"]))
    assert np.array_equal(A.row_offsets, d["A0_ro"]) and np.array_equal(bits(A.values), bits(d["A0_v"]))
    cfg = M.SetupConfig(alpha=float(d["alpha"]), coarse_size_max=40, reuse_caches=True)
    h = backend.setup_hierarchy(A, None, cfg)
    assert h.n_levels() == int(d["n_levels"])
    for k, lvl in enumerate(h.levels):
        Ak = lvl.A
        np.testing.assert_array_equal(Ak.row_offsets, d[f"A{k}_ro"])
        np.testing.assert_array_equal(Ak.col_indices, d[f"A{k}_ci"])
        np.testing.assert_array_equal(bits(Ak.values), bits(d[f"A{k}_v"]))
        np.testing.assert_array_equal(bits(lvl.B), bits(d[f"B{k}"]))
        if k < h.coarsest():
            Pk = lvl.P
            np.testing.assert_array_equal(Pk.col_indices, d[f"P{k}_ci"])
            np.testing.assert_array_equal(bits(Pk.values), bits(d[f"P{k}_v"]))
            om = lvl.smoother.omega
            assert abs(om - float(d[f"omega{k}"])) <= 1e-12 * abs(om)
    method = int(d["method"])
    sc = M.SolverConfig(method=method, tol=1e-8, max_iters=300, restart=30)
    fn = backend.pcg if method == M.PCG else backend.fgmres
    res = fn(A, np.ones(A.n_rows), None, h, M.CycleConfig(), sc)
    hist, want = np.array(res.report.residual_history), d["history"]
    assert hist.shape == want.shape, (hist.shape, want.shape)
    if exact_solve:
        np.testing.assert_array_equal(bits(hist), bits(want))
        np.testing.assert_array_equal(bits(res.x), bits(d["x"]))
    else:
        assert np.max(np.abs(hist - want)) <= 1e-10 * want[0]
        assert np.linalg.norm(res.x - d["x"]) <= 1e-10 * np.linalg.norm(d["x"])
    return res
