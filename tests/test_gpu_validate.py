"""Input validation of the host CSR at the boundary (sparse.cpp:22-39 messages), for small
inputs and for inputs large enough to go through the pinned staging ring, where indices are
narrowed to int32 on the host while being staged (range checks ride along; ordering checks
run on the device)."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

pytestmark = pytest.mark.gpu


def _spmv(gpu, A):
    # setup_hierarchy validates its input, as the reference does (hierarchy.cpp:35)
    return gpu.setup_hierarchy(A, None, M.SetupConfig(coarse_size_max=100))


@pytest.mark.parametrize("n", [50, 700_000])  # 700k rows x 7: > 8 MB of indices (staged)
def test_column_out_of_range_reports_its_row(gpu, n):
    A = gpu.generate_poisson(2, n // 100, 100) if n > 1000 else gpu.generate_poisson(2, 10, 5)
    bad_row = A.n_rows // 2 + 3
    k = A.row_offsets[bad_row] + 1
    A.col_indices[k] = A.n_cols + 5
    with pytest.raises(M.Error, match=f"column index out of range in row {bad_row}"):
        _spmv(gpu, A)
    A.col_indices[k] = -1
    with pytest.raises(M.Error, match=f"column index out of range in row {bad_row}"):
        _spmv(gpu, A)


@pytest.mark.parametrize("n", [50, 700_000])
def test_columns_must_increase(gpu, n):
    A = gpu.generate_poisson(2, n // 100, 100) if n > 1000 else gpu.generate_poisson(2, 10, 5)
    bad_row = A.n_rows - 7
    lo = A.row_offsets[bad_row]
    A.col_indices[lo], A.col_indices[lo + 1] = A.col_indices[lo + 1], A.col_indices[lo]
    with pytest.raises(M.Error, match=f"strictly increasing in row {bad_row}"):
        _spmv(gpu, A)


def test_row_offsets_checks(gpu):
    A = gpu.generate_poisson(2, 600, 1200)  # staged row offsets too
    B = M.SparseMatrix(A.n_rows, A.n_cols, A.row_offsets.copy(), A.col_indices, A.values)
    B.row_offsets[1000] = B.row_offsets[1002]  # decreasing at row 1001
    with pytest.raises(M.Error, match="non-decreasing|strictly increasing"):
        _spmv(gpu, B)


def test_valid_staged_upload_round_trips(gpu, ref):
    A = gpu.generate_poisson(3, 96, 96, 96)  # 6.4 M nnz: staged
    x = np.random.default_rng(3).uniform(-1, 1, A.n_rows)
    y = gpu.spmv(A, x)
    assert np.array_equal(y.view(np.uint64), ref.spmv(A, x).view(np.uint64))
