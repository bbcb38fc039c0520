"""Test configuration.  `-m gpu` tests need a B200 and the built sm_100a library; the
rest run on CPU (oracle vs reference vs golden fixtures, ABI surface, host logic)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 GPU and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def gpu():
    from paper_1403_1649_b200 import aggmg

    b = aggmg.b200()  # raises LibraryMissing loudly if the CUDA library is not built
    rc = b.lib.fn("init")(0)
    if rc != 0:
        raise RuntimeError("aggmg_init failed: " + b.lib.fn("last_error")().decode())
    return b


@pytest.fixture(scope="session")
def ref():
    from paper_1403_1649_b200 import aggmg

    from oracle import checkers

    return checkers.ref()


@pytest.fixture(scope="session")
def orc():
    from paper_1403_1649_b200 import aggmg

    from oracle import checkers

    return checkers.oracle()
