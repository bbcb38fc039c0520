"""CPU: the exact sequential-sum emulation used by the reference-order reductions
(seq_sum_warp in csrc/chunked.cuh, modelled in tools/seqsum_model.py) reproduces the plain
sequential fp64 loop bit for bit on adversarial inputs: ties, cancellation through zero,
binade crossings, subnormals, infinities and NaNs."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import seqsum_model  # noqa: E402


def test_seqsum_model_bit_exact():
    assert seqsum_model.main(40) == 0
