"""The B200 path against the golden fixtures generated from the unmodified reference
(tests/golden/make_golden.py): hierarchies bit-identical, solves within 1e-10 of the
initial residual with equal iteration counts."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

import golden_util as G
from helpers import assert_csr_bits

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", G.HIERARCHY_CASES)
def test_gpu_matches_golden_hierarchy(gpu, name):
    G.check_hierarchy(gpu, name, exact_solve=False)


def test_gpu_worked_example(gpu):
    d = G.load("worked_example")
    A = G.csr(d, "A")
    agg = M.Aggregation(8, 3, d["assignment"], np.array([1, 0, 2]))
    c = gpu.build_galerkin_cache(A, agg)
    for f in ("entry", "entry_row", "segment_offsets", "slot_of_csr"):
        np.testing.assert_array_equal(getattr(c, f), d[f])
    P = M.SparseMatrix(8, 3, np.arange(9), d["assignment"], np.ones(8))
    assert_csr_bits(gpu.apply_galerkin_cache(c, A, P), G.csr(d, "Ac"))


def test_gpu_mis2_golden(gpu):
    d = G.load("mis2_grid")
    S = G.csr(d, "S")
    for key in [k for k in d if k.startswith("state_")]:
        np.testing.assert_array_equal(gpu.mis2(S, d["influence"], int(key[6:])).state, d[key])
