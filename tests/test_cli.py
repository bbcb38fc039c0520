"""The reference command line (aggmg_main.cpp: generate / solve / bench) rebuilt over the
drop-in header as build/aggmg (tools/aggmg_cli.cpp).  CPU: `generate` writes the same bytes
as the reference's own writer, and option errors exit with the reference's input-error code.
GPU: `solve` with the JSON report and run manifest, `--from-manifest` re-runs, the
no-convergence exit code, and the `bench` sweep."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "aggmg")


def run(*args, cwd=None):
    assert os.path.exists(EXE), "build/aggmg missing: run make"
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=600, cwd=cwd)


def test_generate_matches_reference_writer(tmp_path):
    from oracle.checkers import have_ref, ref

    out = run("generate", "--kind", "poisson3d", "--nx", "9", "--ny", "7", "--nz", "5",
              "--epsilon", "0.01", "--matrix-out", str(tmp_path / "A.mtx"),
              "--rhs-out", str(tmp_path / "b.mtx"))
    assert out.returncode == 0, out.stderr
    assert "315 unknowns" in out.stdout
    if have_ref():
        r = ref()
        A = r.generate_poisson(3, 9, 7, 5, 0.01)
        r.write_matrix_market(str(tmp_path / "A_ref.mtx"), A)
        assert (tmp_path / "A.mtx").read_bytes() == (tmp_path / "A_ref.mtx").read_bytes()


def test_option_errors_exit_3():
    assert run("solve", "--bogus").returncode == 3
    assert run("solve", "--solver", "cg").returncode == 3
    assert run("frobnicate").returncode == 3
    assert run("--help").returncode == 0


@pytest.mark.gpu
def test_solve_report_manifest_and_rerun(tmp_path):
    assert run("generate", "--kind", "poisson2d", "--nx", "96", "--ny", "96", "--epsilon", "1",
               "--matrix-out", "A.mtx", "--rhs-out", "b.mtx", cwd=tmp_path).returncode == 0
    out = run("solve", "--matrix", "A.mtx", "--rhs", "b.mtx", "--solver", "pcg", "--tol", "1e-8",
              "--reuse-cache", "--report", "rep.json", "--manifest-out", "man.json", cwd=tmp_path)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "converged in" in out.stdout and "operator complexity" in out.stdout
    rep = json.loads((tmp_path / "rep.json").read_text())
    assert rep["converged"] and rep["iterations"] == len(rep["residual_history"]) - 1
    assert rep["final_relative_residual"] <= 1e-8
    assert rep["manifest"]["config"]["solver"] == "pcg"
    assert rep["manifest"]["inputs"]["matrix"]["hash"].startswith("fnv1a64:")
    # the reference's own solve of the same system: iteration count and history agree
    from oracle.checkers import ref
    from paper_1403_1649_b200 import aggmg as M

    r = ref()
    A = r.read_matrix_market(str(tmp_path / "A.mtx"))
    h = r.setup_hierarchy(A, None, M.SetupConfig(reuse_caches=True))
    rr = r.pcg(A, r.read_vector_market(str(tmp_path / "b.mtx")), None, h, M.CycleConfig(),
               M.SolverConfig(method=M.PCG, tol=1e-8, max_iters=200))
    assert rr.report.iterations == rep["iterations"]
    hr = np.array(rr.report.residual_history)
    assert np.max(np.abs(np.array(rep["residual_history"]) - hr)) <= 1e-10 * hr.max()
    # --from-manifest reproduces the run
    again = run("solve", "--from-manifest", "man.json", "--report", "rep2.json", cwd=tmp_path)
    assert again.returncode == 0, again.stderr
    assert json.loads((tmp_path / "rep2.json").read_text())["iterations"] == rep["iterations"]
    # no convergence -> exit code 2
    assert run("solve", "--matrix", "A.mtx", "--max-iters", "2", "--tol", "1e-12",
               cwd=tmp_path).returncode == 2


@pytest.mark.gpu
def test_bench_sweep(tmp_path):
    out = run("bench", "--sizes", "32,64", "--solver", "pcg", "--tol", "1e-8",
              "--galerkin-refresh", "64", "--out", "b.json", cwd=tmp_path)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads((tmp_path / "b.json").read_text())
    assert [row["size"] for row in res["rows"]] == [32, 64]
    assert all(row["converged"] for row in res["rows"])
    assert res["galerkin_refresh"]["size"] == 64
