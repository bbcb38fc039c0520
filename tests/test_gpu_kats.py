"""The reference's own known-answer tests (SURVEY §8c parity pins), re-run on the B200
library: the same functions test_oracle.py applies to the C restatement, called with the
device backend.  Ties at the strength threshold, MIS(2) on isolated nodes / paths / stars and
its distance-2 independence + maximality on seeded random graphs, the pass-2 weight and
tie-break rule, transfer hand values, omega == 4/3 on diagonal matrices, the Eq. 8 worked
example's exact power-of-two sums."""
import pytest

import test_oracle as K

pytestmark = pytest.mark.gpu


def test_worked_example_exact_sums(gpu):
    K.test_worked_example_exact_sums(gpu)


def test_strength_hand_cases(gpu):
    K.test_strength_hand_cases(gpu)


def test_mis2_small_graphs(gpu):
    K.test_mis2_small_graphs(gpu)


def test_mis2_bfs_properties(gpu):
    K.test_mis2_bfs_properties(gpu)


def test_pass2_tie_break(gpu):
    K.test_pass2_tie_break(gpu)


def test_transfer_hand_case(gpu):
    K.test_transfer_hand_case(gpu)


def test_omega_diagonal_exact(gpu):
    K.test_omega_diagonal_exact(gpu)
