"""Full-size parity at the BASELINE configurations (size-independent properties + the
reference's own full-size facts).

The reference was run at full size during the survey ("Measured here": 8-core
Xeon, seed 42, b = B0 = ones, x0 = 0, hybrid K-cycle): its level sizes and outer iteration
counts are pinned below for both Galerkin paths.  The device hierarchy must reproduce the level
sizes exactly (they are a function of every aggregate at every level) and the iteration count;
the final TRUE residual must meet the tolerance (a solve-independent check)."""
import ctypes as C

import numpy as np
import pytest

from paper_1403_1649_b200 import _abi
from paper_1403_1649_b200 import aggmg as M
from paper_1403_1649_b200 import dist as D

pytestmark = pytest.mark.gpu

# (dims, n, eps, method, reuse_caches) -> (level sizes, iterations)
REFERENCE = {
    (3, 128, 1.0, "pcg", True): ([2097152, 189710, 18419, 1641, 149], 30),
    (3, 128, 1.0, "pcg", False): ([2097152, 189710, 18608, 1620, 155], 30),
    (3, 256, 1.0, "pcg", True): ([16777216, 1505380, 143921, 12402, 1080, 103], 42),
    (3, 256, 1.0, "pcg", False): ([16777216, 1505380, 145490, 12558, 1094, 101], 42),
    (3, 384, 1e-3, "fgmres", True): ([56623104, 7952102, 1029806, 136911, 19084, 3055, 541], 63),
    (3, 384, 1e-3, "fgmres", False): ([56623104, 7952102, 1029806, 136929, 19191, 3089, 562], 65),
    (2, 512, 1.0, "pcg", False): ([262144, 36791, 3713, 367], 33),
}


def _check(rc, lib):
    assert rc == 0, lib.fn("last_error")().decode()


@pytest.mark.parametrize("key", list(REFERENCE), ids=lambda k: f"{k[0]}d-{k[1]}-eps{k[2]}-{k[3]}-"
                                                              f"{'cache' if k[4] else 'direct'}")
def test_full_size_levels_and_iterations(gpu, key):
    dims, n, eps, method, cache = key
    sizes, its = REFERENCE[key]
    lib = gpu.lib
    dm = C.c_void_p()
    _check(lib.fn("dmatrix_poisson")(dims, n, n, n if dims == 3 else 1, eps, -1, C.byref(dm)), lib)
    cfg = M.SetupConfig(alpha=0.5 if dims == 3 else 0.25, reuse_caches=cache)._c()
    h = C.c_void_p()
    _check(lib.fn("setup_hierarchy_device")(dm, C.byref(cfg), C.byref(h)), lib)
    got = []
    for k in range(lib.fn("hierarchy_n_levels")(h)):
        nk, nnz = C.c_int64(), C.c_int64()
        _check(lib.fn("hierarchy_level_size")(h, k, C.byref(nk), C.byref(nnz)), lib)
        got.append(nk.value)
    assert got == sizes
    sc = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=1e-8, max_iters=500,
                        restart=30)._c()
    cc = M.CycleConfig()._c()
    rep = _abi.SolveReportC()
    hist = np.zeros(600)
    rep.history = hist.ctypes.data_as(_abi.f64p)
    rep.history_capacity = hist.shape[0]
    nn = sizes[0]
    x = np.zeros(nn)
    _check(lib.fn("solve_device")(h, C.byref(cc), C.byref(sc), x.ctypes.data_as(_abi.f64p),
                                  C.byref(rep)), lib)
    assert rep.converged and rep.iterations == its
    lib.fn("hierarchy_free")(h)
    if nn > 20_000_000:  # 384^3: level sizes and the iteration count only (host memory)
        lib.fn("dmatrix_free")(dm)
        return
    # the true residual ||b - A x|| / ||b|| of the returned solution (b = ones)
    out = _abi.CSR()
    _check(lib.fn("dmatrix_to_host")(dm, C.byref(out)), lib)
    try:
        ro = np.ctypeslib.as_array(out.row_offsets, shape=(nn + 1,))
        ci = np.ctypeslib.as_array(out.col_indices, shape=(out.nnz,))
        va = np.ctypeslib.as_array(out.values, shape=(out.nnz,))
        Ax = np.add.reduceat(va * x[ci], ro[:-1])
        rel = np.linalg.norm(1.0 - Ax) / np.sqrt(nn)
    finally:
        lib.fn("csr_free")(C.byref(out))
        lib.fn("dmatrix_free")(dm)
    assert rel <= 1.5e-8, rel


def test_full_size_partitioned_levels(gpu):
    """256^3 on 2 rank threads: the same hierarchy (level sizes) and iteration count."""
    sizes, its = REFERENCE[(3, 256, 1.0, "pcg", True)]
    out = {}

    def fn(comm, r):
        A = D.DistMatrix.poisson(comm, 3, 256, 256, 256)
        h = D.setup(comm, A, M.SetupConfig(alpha=0.5, reuse_caches=True))
        out[r] = ([h.level_size(k)[0] for k in range(h.n_levels())], h.info()[1],
                  h.solve(M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=500)).report)
        h.free()
        A.free()

    D.run_threads(2, fn)
    got, nd, rep = out[0]
    assert got == sizes and nd >= 1
    assert rep.converged and rep.iterations == its
