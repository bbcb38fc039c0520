"""pcg / fgmres with an arbitrary host preconditioner (the reference's std::function
Preconditioner, krylov.hpp:38): the device Krylov loop calls back once per application.
Compared with the reference's own solvers driven by the same callable."""
import numpy as np
import pytest

from paper_1403_1649_b200 import aggmg as M

from helpers import bits, random_spd

pytestmark = pytest.mark.gpu


def _jacobi(A):
    d = A.values[np.repeat(np.arange(A.n_rows), np.diff(A.row_offsets)) == A.col_indices]
    return lambda r: r / d


@pytest.mark.parametrize("method", ["pcg", "fgmres"])
def test_jacobi_callback_matches_reference(gpu, ref, method):
    for A in (random_spd(300, 0.05, 21), ref.generate_poisson(2, 64, 64)):
        b = np.linspace(-1.0, 1.0, A.n_rows)
        cfg = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=1e-8,
                             max_iters=600, restart=60)
        rg = getattr(gpu, method)(A, b, None, _jacobi(A), None, cfg)
        rr = getattr(ref, method)(A, b, None, _jacobi(A), None, cfg)
        assert rg.report.converged == rr.report.converged
        assert rg.report.iterations == rr.report.iterations
        hg, hr = np.array(rg.report.residual_history), np.array(rr.report.residual_history)
        assert np.max(np.abs(hg - hr)) <= 1e-10 * hr[0]
        # with the reference's reduction order the whole solve is bit-identical
        gpu.lib.fn("set_exact_reductions")(1)
        try:
            re = getattr(gpu, method)(A, b, None, _jacobi(A), None, cfg)
        finally:
            gpu.lib.fn("set_exact_reductions")(0)
        np.testing.assert_array_equal(bits(np.array(re.report.residual_history)), bits(hr))
        np.testing.assert_array_equal(bits(re.x), bits(rr.x))


def test_amg_lambda_equals_device_cycle(gpu):
    """The CLI's wiring (aggmg_main.cpp:194-196): a lambda around apply_preconditioner."""
    A = gpu.generate_poisson(2, 128, 128)
    cfg = M.SetupConfig(reuse_caches=True)
    h = gpu.setup_hierarchy(A, None, cfg)
    cc = M.CycleConfig()
    sc = M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200)
    b = np.ones(A.n_rows)
    lam = gpu.pcg(A, b, None, lambda r: gpu.apply_preconditioner(h, cc, r), cc, sc)
    dev = gpu.pcg(A, b, None, h, cc, sc)
    assert lam.report.iterations == dev.report.iterations
    hl, hd = np.array(lam.report.residual_history), np.array(dev.report.residual_history)
    assert np.max(np.abs(hl - hd)) <= 1e-12 * hd[0]


def test_callback_errors_propagate(gpu):
    A = random_spd(50, 0.1, 3)

    def bad(r):
        raise ValueError("boom")

    with pytest.raises(ValueError, match="boom"):
        gpu.pcg(A, np.ones(50), None, bad, None, M.SolverConfig(method=M.PCG))
    with pytest.raises(M.Error, match="length"):
        gpu.fgmres(A, np.ones(50), None, lambda r: r[:10], None, M.SolverConfig())
