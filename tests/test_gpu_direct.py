"""The reference's DEFAULT coarse-operator path (reuse_caches = false: galerkin_direct =
spmm(spmm(R, A), P), galerkin.cpp:33-36) on the device: bit-identical coarse values and
therefore bit-identical hierarchies for default-config callers, including 3-D problems
where the two reference paths diverge."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

import golden_util as G
from helpers import assert_csr_bits, bits, random_sparse, random_spd

pytestmark = pytest.mark.gpu


def test_galerkin_direct_bit_exact(gpu, ref):
    rng = np.random.default_rng(17)
    for seed in range(6):
        n = 50 + 23 * seed
        nc = 2 + 3 * seed
        A = random_sparse(n, n, 0.12, 300 + seed)
        a = np.concatenate([np.arange(nc), rng.integers(0, nc, n - nc)]).astype(np.int64)
        agg = M.Aggregation(n, nc, a, np.zeros(nc, dtype=np.int64))
        b = rng.uniform(0.2, 2.0, n)
        if seed % 2:
            b[::7] = 0.0  # empty P rows / R columns
            if any(np.all(b[a == J] == 0) for J in range(nc)):
                continue
        t = ref.build_transfer(agg, b)
        assert_csr_bits(gpu.galerkin_direct(t.R, A, t.P), ref.galerkin_direct(t.R, A, t.P))


def test_galerkin_direct_long_rows(gpu, ref):
    A = random_spd(600, 0.02, 8)
    agg = M.Aggregation(600, 2, (np.arange(600) % 2).astype(np.int64), np.array([0, 1]))
    t = ref.build_transfer(agg, np.ones(600))
    assert_csr_bits(gpu.galerkin_direct(t.R, A, t.P), ref.galerkin_direct(t.R, A, t.P))


def test_worked_example_direct(gpu):
    d = G.load("worked_example")
    A = G.csr(d, "A")
    P = M.SparseMatrix(8, 3, np.arange(9), d["assignment"], np.ones(8))
    Ac = gpu.galerkin_direct(gpu.transpose(P), A, P)
    assert list(Ac.row_offsets) == [0, 3, 5, 7]
    assert list(Ac.col_indices) == [0, 1, 2, 0, 1, 0, 2]
    np.testing.assert_array_equal(bits(Ac.values), bits(G.csr(d, "Ac").values))


@pytest.mark.parametrize("case", ["2d-96", "3d-28", "3d-aniso-24"])
def test_default_config_hierarchy_bit_exact(gpu, ref, case):
    A, alpha = {
        "2d-96": (ref.generate_poisson(2, 96, 96), 0.25),
        "3d-28": (ref.generate_poisson(3, 28, 28, 28), 0.5),
        "3d-aniso-24": (ref.generate_poisson(3, 24, 24, 24, 1e-3), 0.5),
    }[case]
    cfg = M.SetupConfig(alpha=alpha, coarse_size_max=40)  # reuse_caches = False (default)
    hg, hr = gpu.setup_hierarchy(A, None, cfg), ref.setup_hierarchy(A, None, cfg)
    assert hg.n_levels() == hr.n_levels()
    for k, (lg, lr) in enumerate(zip(hg.levels, hr.levels)):
        assert_csr_bits(lg.A, lr.A, f"A level {k}")
        if k < hg.coarsest():
            assert_csr_bits(lg.P, lr.P, f"P level {k}")
            assert lg.smoother.omega == lr.smoother.omega
