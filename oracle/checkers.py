"""TEST INFRASTRUCTURE — the CPU checkers behind the product's Python binding.

Only tests/, __graft_entry__.smoke(), bench.py's cpu_baseline / --impl reference legs and
tools/ import this module.  The product package (paper_1403_1649_b200) never loads these
libraries; they are the yardsticks the CUDA path is compared against:

    oracle()  oracle/liboracle.so          — the C restatement (aggmg_oracle.c), every
                                            function citing the reference file:line it follows
    ref()     oracle/_ref/libaggmg_ref.so  — the UNMODIFIED reference sources
                                            (/root/reference/proj/core/src) compiled by
                                            oracle/Makefile behind the shim ref_shim.cpp

Both export the same C interface as the product (include/aggmg_b200.h) under their own
prefixes, so the product's Backend class drives them unchanged.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
if REPO not in sys.path:
    sys.path.insert(0, REPO)

from paper_1403_1649_b200 import _abi  # noqa: E402
from paper_1403_1649_b200.aggmg import Backend  # noqa: E402

ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libaggmg_ref.so")

_cache = {}


def _get(name, path, prefix):
    b = _cache.get(name)
    if b is None:
        b = _cache[name] = Backend(_abi.Lib(path, prefix), name)
    return b


def oracle() -> Backend:
    """The C restatement in oracle/ (aggmg_oracle.c)."""
    return _get("oracle", ORACLE_LIB, "aggmg_oracle_")


def ref() -> Backend:
    """The unmodified reference compiled into oracle/_ref/."""
    return _get("ref", REF_LIB, "aggmg_ref_")


def have_ref() -> bool:
    return os.path.exists(REF_LIB)
