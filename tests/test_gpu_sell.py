"""The SELL-32 kernel family (large square operators with 4-64 entries per row): bit-exact
against the reference SpMV, and kept consistent when refresh_values rewrites the values.
The matrices here pass the SELL threshold (>= 2^19 rows); the other parity tests run the
CSR-stream kernel."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import bits

pytestmark = pytest.mark.gpu


def banded_irregular(n, seed):
    """Rows of 8-24 distinct sorted columns within +-600 of the diagonal (diagonal included)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(8, 25, n)
    rows, cols = [], []
    for lo in range(0, n, 65536):
        hi = min(n, lo + 65536)
        r = np.repeat(np.arange(lo, hi), lens[lo:hi])
        c = np.clip(r + rng.integers(-600, 601, r.shape[0]), 0, n - 1)
        rows.append(np.concatenate([r, np.arange(lo, hi)]))
        cols.append(np.concatenate([c, np.arange(lo, hi)]))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    ro = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ro, r + 1, 1)
    v = rng.uniform(-1, 1, key.shape[0])
    return M.SparseMatrix(n, n, np.cumsum(ro), c, v)


def test_sell_spmv_bit_exact(gpu, ref):
    rng = np.random.default_rng(3)
    for A in (gpu.generate_jump27(82, 82, 82, 1e6, 32), banded_irregular(600_000, 7),
              gpu.generate_poisson(3, 82, 82, 82)):
        assert A.n_rows >= 1 << 19 and A.col_indices.shape[0] >= 4 * A.n_rows
        x = rng.uniform(-1, 1, A.n_cols)
        np.testing.assert_array_equal(bits(gpu.spmv(A, x)), bits(ref.spmv(A, x)))


def test_sell_refresh_values(gpu):
    # a refreshed hierarchy must solve exactly like one set up on the new values
    A = gpu.generate_jump27(82, 82, 82, 1e6, 32)
    A2 = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, A.values * 3.0)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    b = np.ones(A.n_rows)
    h = gpu.setup_hierarchy(A, None, cfg)
    gpu.refresh_values(h, A2.values)
    r1 = gpu.pcg(A2, b, None, h, M.CycleConfig(), sc)
    r2 = gpu.pcg(A2, b, None, gpu.setup_hierarchy(A2, None, cfg), M.CycleConfig(), sc)
    assert r1.report.iterations == r2.report.iterations
    np.testing.assert_array_equal(bits(np.array(r1.report.residual_history)),
                                  bits(np.array(r2.report.residual_history)))


def test_sell_arnoldi_omega_bit_exact(gpu, ref):
    # the damped-Jacobi Arnoldi estimate runs its SpMVs through the SELL-32 kernel on operators
    # this large; omega and rho stay bit-identical to the reference
    A = gpu.generate_poisson(3, 104, 104, 104)
    sg = gpu.setup_smoother(A, M.DAMPED_JACOBI, 5, 11)
    sr = ref.setup_smoother(A, M.DAMPED_JACOBI, 5, 11)
    assert sg.omega == sr.omega and sg.rho_est == sr.rho_est
    np.testing.assert_array_equal(bits(sg.inv_diag), bits(sr.inv_diag))


def _dmatrix_format(gpu, A):
    """aggmg_dmatrix_format of A uploaded as a device matrix: 0 CSR, 1 SELL, 2 SELL + dictionary,
    3 row patterns."""
    import ctypes as C
    lib = gpu.lib
    dm = C.c_void_p()
    csr = A._c()
    assert lib.fn("dmatrix_from_host")(C.byref(csr), C.byref(dm)) == 0, lib.fn("last_error")().decode()
    f = C.c_int32()
    assert lib.fn("dmatrix_format")(dm, C.byref(f)) == 0
    lib.fn("dmatrix_free")(dm)
    return f.value


@pytest.mark.parametrize("distinct", [1, 2, 256, 257])
def test_sell_value_dictionary_bit_exact(gpu, ref, distinct):
    # <= 256 distinct values: SELL stores one-byte codes into a value table; 257: plain SELL.
    # Either way the SpMV is bit-identical to the reference.
    A = gpu.generate_poisson(3, 82, 82, 82)
    rng = np.random.default_rng(distinct)
    table = rng.uniform(-2, 2, distinct)
    table[0] = -0.0  # signed zero is its own pattern
    codes = rng.integers(0, distinct, A.values.shape[0])
    codes[:distinct] = np.arange(distinct)  # every value occurs
    B = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, table[codes])
    x = rng.uniform(-1, 1, A.n_cols)
    np.testing.assert_array_equal(bits(gpu.spmv(B, x)), bits(ref.spmv(B, x)))
    # few distinct values: the rows repeat at most a few thousand patterns (format 3)
    assert _dmatrix_format(gpu, B) in {1: (3,), 2: (2, 3), 256: (2,), 257: (1,)}[distinct]


def test_sell_value_dictionary_refresh(gpu):
    # refresh_values that leaves the dictionary range (random values) and comes back
    A = gpu.generate_poisson(3, 82, 82, 82)
    rng = np.random.default_rng(5)
    v = A.values.copy()  # random diagonal shifts: SPD, thousands of distinct values
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    diag = A.col_indices == rows
    v[diag] += rng.uniform(0.0, 1.0, int(diag.sum()))
    A_rand = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, v)
    assert _dmatrix_format(gpu, A_rand) == 1 and _dmatrix_format(gpu, A) == 3
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    b = np.ones(A.n_rows)
    h = gpu.setup_hierarchy(A, None, cfg)
    for B in (A_rand, A):
        gpu.refresh_values(h, B.values)
        r1 = gpu.pcg(B, b, None, h, M.CycleConfig(), sc)
        r2 = gpu.pcg(B, b, None, gpu.setup_hierarchy(B, None, cfg), M.CycleConfig(), sc)
        assert r1.report.iterations == r2.report.iterations
        np.testing.assert_array_equal(bits(np.array(r1.report.residual_history)),
                                      bits(np.array(r2.report.residual_history)))
