"""B200-native unsmoothed-aggregation AMG (arXiv 1403.1649), drop-in for the reference
`aggmg` setup/solve path.  The compute path is the sm_100a library
paper_1403_1649_b200/lib/libaggmg_b200.so behind the C-ABI in include/aggmg_b200.h;
this package is the Python binding of that boundary (see aggmg.py)."""
from .aggmg import (  # noqa: F401
    CYCLE_HYBRID, CYCLE_K, CYCLE_V, DAMPED_JACOBI, FGMRES, INNER_CG, INNER_GMRES, JACOBI, PCG,
    SGS, Aggregation, CycleConfig, Error, CudaError, Hierarchy, Mis2Result, SetupConfig,
    SolverConfig, SparseMatrix, b200, ones_vector)

__version__ = "0.1.0"
