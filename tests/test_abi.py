"""CPU checks of the drop-in boundary: the built sm_100a library loads and exports every
entry point include/aggmg_b200.h declares; the ctypes table covers the header; the
reference shim exports the same names (no compute calls: no GPU here)."""
import os
import re
import subprocess

import pytest

from paper_1403_1649_b200 import _abi

HEADER = os.path.join(_abi.REPO, "include", "aggmg_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(aggmg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_surface():
    names = declared()
    for must in ("aggmg_setup_hierarchy", "aggmg_apply_preconditioner", "aggmg_pcg",
                 "aggmg_fgmres", "aggmg_classic_strength", "aggmg_mis2", "aggmg_aggregate",
                 "aggmg_build_transfer", "aggmg_build_galerkin_cache",
                 "aggmg_apply_galerkin_cache", "aggmg_setup_smoother", "aggmg_smooth",
                 "aggmg_spmv", "aggmg_vcycle", "aggmg_kcycle", "aggmg_refresh_values"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _abi.Lib(_abi.PRODUCT_LIB, "aggmg_")
    missing = [n for n in declared() if not lib.has(n[len("aggmg_"):])]
    assert not missing, missing


def test_ctypes_table_covers_header():
    names = {n[len("aggmg_"):] for n in declared()}
    assert names <= set(_abi.SIGNATURES), sorted(names - set(_abi.SIGNATURES))


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _abi.PRODUCT_LIB],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_reference_shim_exports_same_names():
    from oracle.checkers import REF_LIB

    if not os.path.exists(REF_LIB):
        pytest.skip("reference shim not built")
    lib = _abi.Lib(REF_LIB, "aggmg_ref_")
    shared = ["setup_hierarchy", "apply_preconditioner", "pcg", "fgmres", "classic_strength",
              "mis2", "aggregate", "build_transfer", "build_galerkin_cache",
              "apply_galerkin_cache", "setup_smoother", "smooth", "spmv", "vcycle", "kcycle"]
    assert all(lib.has(n) for n in shared)


def test_no_gpu_call_fails_loudly():
    """Without a GPU the product must refuse, not fall back to the CPU."""
    import ctypes

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    lib = _abi.Lib(_abi.PRODUCT_LIB, "aggmg_")
    rc = lib.fn("init")(0)
    assert rc == 2
    assert b"CUDA" in lib.fn("last_error")() or b"device" in lib.fn("last_error")()
    _ = ctypes
