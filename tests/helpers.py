"""Shared generators and comparators for the parity tests (mirrors the role of the
reference's tests/support/test_helpers.hpp: seeded generators, dumb comparators)."""
import numpy as np

from paper_1403_1649_b200.aggmg import SparseMatrix


def from_triplets(n, m, rows, cols, vals):
    rows, cols, vals = np.asarray(rows), np.asarray(cols), np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    key = rows * m + cols
    uniq, start = np.unique(key, return_index=True)
    sums = np.add.reduceat(vals, start) if len(vals) else vals
    r, c = uniq // m, uniq % m
    ro = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ro, r + 1, 1)
    return SparseMatrix(n, m, np.cumsum(ro), c, sums)


def random_sparse(n, m, density, seed):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, m)) < density
    r, c = np.nonzero(mask)
    return from_triplets(n, m, r, c, rng.uniform(-1, 1, r.shape[0]))


def random_spd(n, density, seed):
    rng = np.random.default_rng(seed)
    up = np.triu(rng.random((n, n)) < density, 1)
    r, c = np.nonzero(up)
    v = rng.uniform(-1, 1, r.shape[0])
    rows = np.concatenate([r, c, np.arange(n)])
    cols = np.concatenate([c, r, np.arange(n)])
    rowsum = np.zeros(n)
    np.add.at(rowsum, r, np.abs(v))
    np.add.at(rowsum, c, np.abs(v))
    vals = np.concatenate([v, v, rowsum + 1.0])
    return from_triplets(n, n, rows, cols, vals)


def random_graph(n, density, seed):
    rng = np.random.default_rng(seed)
    up = np.triu(rng.random((n, n)) < density, 1)
    r, c = np.nonzero(up)
    return from_triplets(n, n, np.concatenate([r, c]), np.concatenate([c, r]),
                         np.ones(2 * r.shape[0]))


def laplacian_1d(n):
    i = np.arange(n)
    rows = np.concatenate([i[1:], i, i[:-1]])
    cols = np.concatenate([i[:-1], i, i[1:]])
    vals = np.concatenate([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)])
    return from_triplets(n, n, rows, cols, vals)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_csr_bits(A, B, what=""):
    assert A.n_rows == B.n_rows and A.n_cols == B.n_cols, what
    np.testing.assert_array_equal(A.row_offsets, B.row_offsets, err_msg=what)
    np.testing.assert_array_equal(A.col_indices, B.col_indices, err_msg=what)
    np.testing.assert_array_equal(bits(A.values), bits(B.values), err_msg=what)


def assert_pattern(A, B, what=""):
    assert A.n_rows == B.n_rows and A.n_cols == B.n_cols, what
    np.testing.assert_array_equal(A.row_offsets, B.row_offsets, err_msg=what)
    np.testing.assert_array_equal(A.col_indices, B.col_indices, err_msg=what)


def max_rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    scale = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)
    return float(np.max(np.abs(a - b) / scale)) if a.size else 0.0


def rel_norm(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(a - b)
    s = max(np.linalg.norm(a), np.linalg.norm(b), 1e-300)
    return float(d / s)
