"""The drop-in C++ API (include/aggmg/aggmg.hpp) driven by a reference-style caller
(tools/cpp_dropin_demo.cpp, built by `make`): the reference's acceptance criteria for
sparsity, grid independence, refresh and run-to-run determinism, the CLI's lambda preconditioner
(aggmg_main.cpp:194-200), the Jacobi-PCG known-answer test (test_krylov.cpp:129-156) and
refresh_values' by-value semantics (hierarchy.cpp:90), on the B200 path."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_acceptance():
    exe = os.path.join(ROOT, "build", "cpp_dropin_demo")
    assert os.path.exists(exe), "build/cpp_dropin_demo missing: run make"
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout and out.stdout.count("PASS") == 8
