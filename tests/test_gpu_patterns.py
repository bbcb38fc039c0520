"""The row-pattern format (sparse.cu build_patterns / k_pat): a stencil operator stored as a
two-byte pattern id per row plus pattern tables of (offset from the diagonal position, value).
Every SpMV epilogue must be bit-identical to the reference and to the SELL-32 copy of the same
operator; refresh_values keeps or drops the format as the new values allow."""
import ctypes as C

import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import bits
from test_gpu_sell import _dmatrix_format

pytestmark = pytest.mark.gpu


def _patterns(gpu, on):
    gpu.lib.fn("set_row_patterns")(1 if on else 0)


@pytest.mark.parametrize("dims", [2, 3])
def test_pattern_spmv_bit_exact(gpu, ref, dims):
    n = 760 if dims == 2 else 84  # >= 2^19 rows: the formats of the large operators
    A = gpu.generate_poisson(dims, n, n, n if dims == 3 else 1)
    assert _dmatrix_format(gpu, A) == 3
    rng = np.random.default_rng(dims)
    x = rng.uniform(-1, 1, A.n_cols)
    x[::97] = 0.0
    x[5] = -0.0
    np.testing.assert_array_equal(bits(gpu.spmv(A, x)), bits(ref.spmv(A, x)))


def test_pattern_boundary_rows_and_shifted_values(gpu, ref):
    # a stencil whose diagonal differs on every z-plane: ~ (boundary patterns) x planes
    # distinct rows, still far below the pattern limit
    A = gpu.generate_poisson(3, 90, 90, 90)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    v = A.values.copy()
    diag = A.col_indices == rows
    v[diag] += (rows[diag] // (90 * 90)) * 0.125
    B = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, v)
    assert _dmatrix_format(gpu, B) == 3
    x = np.random.default_rng(3).uniform(-1, 1, B.n_cols)
    np.testing.assert_array_equal(bits(gpu.spmv(B, x)), bits(ref.spmv(B, x)))


def test_too_many_patterns_fall_back(gpu, ref):
    # every row its own diagonal value: more patterns than the format takes, but few enough
    # distinct values for the dictionary -> SELL-32 + dictionary
    A = gpu.generate_poisson(3, 84, 84, 84)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    v = A.values.copy()
    diag = A.col_indices == rows
    v[diag] += (rows[diag] % 200) * 0.01  # 200 diagonal values spread over the grid
    B = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, v)
    assert _dmatrix_format(gpu, B) in (2, 3)
    x = np.random.default_rng(4).uniform(-1, 1, B.n_cols)
    np.testing.assert_array_equal(bits(gpu.spmv(B, x)), bits(ref.spmv(B, x)))


def test_patterns_and_sell_solve_bit_identical(gpu):
    # exact mode: the whole solve through the pattern kernels equals the SELL-32 one bit for bit
    A = gpu.generate_poisson(3, 84, 84, 84)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    b = np.ones(A.n_rows)
    out = []
    gpu.lib.fn("set_exact_reductions")(1)
    try:
        for on in (True, False):
            _patterns(gpu, on)
            h = gpu.setup_hierarchy(A, None, cfg)
            from test_gpu_fullsize_pins import _level_format
            assert _level_format(gpu, h, 0) == (3 if on else 2)
            out.append(gpu.pcg(A, b, None, h, M.CycleConfig(), sc))
    finally:
        gpu.lib.fn("set_exact_reductions")(0)
        _patterns(gpu, True)
    assert out[0].report.iterations == out[1].report.iterations
    np.testing.assert_array_equal(bits(np.array(out[0].report.residual_history)),
                                  bits(np.array(out[1].report.residual_history)))
    np.testing.assert_array_equal(bits(out[0].x), bits(out[1].x))


def test_pattern_refresh(gpu):
    # refresh to scaled stencil values (still patterns), to random values (SELL) and back
    A = gpu.generate_poisson(3, 84, 84, 84)
    cfg = M.SetupConfig(alpha=0.5, reuse_caches=True)
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    b = np.ones(A.n_rows)
    rng = np.random.default_rng(9)
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets))
    v_rand = A.values.copy()
    v_rand[A.col_indices == rows] += rng.uniform(0.0, 1.0, A.n_rows)
    h = gpu.setup_hierarchy(A, None, cfg)
    for vals in (2.0 * A.values, v_rand, A.values):
        B = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets, A.col_indices, vals)
        gpu.refresh_values(h, B.values)
        r1 = gpu.pcg(B, b, None, h, M.CycleConfig(), sc)
        r2 = gpu.pcg(B, b, None, gpu.setup_hierarchy(B, None, cfg), M.CycleConfig(), sc)
        assert r1.report.iterations == r2.report.iterations
        np.testing.assert_array_equal(bits(np.array(r1.report.residual_history)),
                                      bits(np.array(r2.report.residual_history)))
