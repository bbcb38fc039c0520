"""ctypes description of the C-ABI in include/aggmg_b200.h.

The same signature table binds three shared libraries that export the interface
under different prefixes:

  * ``aggmg_``        paper_1403_1649_b200/lib/libaggmg_b200.so — the product (sm_100a kernels)
  * ``aggmg_oracle_`` oracle/liboracle.so — the C restatement (test infrastructure)
  * ``aggmg_ref_``    oracle/_ref/libaggmg_ref.so — the unmodified reference behind a C shim
                      (test infrastructure)
"""
from __future__ import annotations

import ctypes as C
import os

i8p = C.POINTER(C.c_int8)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class CSR(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int64),
        ("n_cols", C.c_int64),
        ("nnz", C.c_int64),
        ("row_offsets", i64p),
        ("col_indices", i64p),
        ("values", f64p),
    ]


class SetupConfigC(C.Structure):
    _fields_ = [
        ("alpha", C.c_double),
        ("coarse_size_max", C.c_int64),
        ("max_levels", C.c_int32),
        ("smoother", C.c_int32),
        ("arnoldi_m", C.c_int32),
        ("reuse_caches", C.c_int32),
        ("seed", C.c_uint64),
    ]


class CycleConfigC(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("k_levels", C.c_int32),
        ("t", C.c_double),
        ("inner", C.c_int32),
    ]


class SolverConfigC(C.Structure):
    _fields_ = [
        ("method", C.c_int32),
        ("tol", C.c_double),
        ("max_iters", C.c_int32),
        ("restart", C.c_int32),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("converged", C.c_int32),
        ("iterations", C.c_int32),
        ("history", f64p),
        ("history_capacity", C.c_int64),
        ("history_length", C.c_int64),
        ("setup_seconds", C.c_double),
        ("solve_seconds", C.c_double),
        ("note", C.c_char * 256),
    ]


csrp = C.POINTER(CSR)
# int (*)(aggmg_comm*, int rank, void* user)
RANK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p)
# aggmg_precond_fn: z = M(r) over host arrays of n doubles
PRECOND_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64,
                         C.c_void_p)
I = C.c_int
L = C.c_int64

# name -> (restype, argtypes).  Opaque handles are void*.
SIGNATURES = {
    "last_error": (C.c_char_p, []),
    "csr_free": (None, [csrp]),
    "spmv": (I, [csrp, f64p, f64p]),
    "transpose": (I, [csrp, csrp]),
    "dot": (I, [L, f64p, f64p, f64p]),
    "norm2": (I, [L, f64p, f64p]),
    "axpy": (I, [L, C.c_double, f64p, f64p]),
    "scale": (I, [L, C.c_double, f64p]),
    "classic_strength": (I, [csrp, C.c_double, I, csrp]),
    "influence_counts": (I, [csrp, i64p]),
    "symmetrize_pattern": (I, [csrp, csrp]),
    "mis2": (I, [csrp, i64p, C.c_uint64, i8p, i64p, i32p]),
    "aggregate": (I, [csrp, csrp, i8p, i64p, i64p, i64p]),
    "build_transfer": (I, [L, L, i64p, f64p, csrp, csrp, f64p]),
    "galerkin_direct": (I, [csrp, csrp, csrp, csrp]),
    "build_galerkin_cache": (I, [csrp, L, i64p, C.POINTER(vp)]),
    "galerkin_cache_info": (I, [vp, i64p, i64p, i64p, i64p]),
    "galerkin_cache_export": (I, [vp, i64p, i64p, i64p, i64p, i64p, i64p, i64p, i64p]),
    "apply_galerkin_cache": (I, [vp, csrp, csrp, csrp]),
    "galerkin_cache_free": (None, [vp]),
    "setup_smoother": (I, [csrp, I, I, C.c_uint64, f64p, f64p, f64p]),
    "smooth": (I, [I, f64p, C.c_double, csrp, f64p, f64p]),
    "hessenberg_eigenvalues": (I, [L, f64p, f64p, f64p]),
    "setup_hierarchy": (I, [csrp, f64p, C.POINTER(SetupConfigC), C.POINTER(vp)]),
    "refresh_values": (I, [vp, f64p, L]),
    "hierarchy_clone": (I, [vp, C.POINTER(vp)]),
    "hierarchy_free": (None, [vp]),
    "hierarchy_n_levels": (L, [vp]),
    "hierarchy_level_size": (I, [vp, L, i64p, i64p]),
    "hierarchy_level_A": (I, [vp, L, csrp]),
    "hierarchy_level_P": (I, [vp, L, csrp]),
    "hierarchy_level_R": (I, [vp, L, csrp]),
    "hierarchy_level_B": (I, [vp, L, f64p]),
    "hierarchy_level_aggregation": (I, [vp, L, i64p, i64p, i32p]),
    "hierarchy_level_smoother": (I, [vp, L, f64p, f64p, f64p]),
    "hierarchy_n_warnings": (L, [vp]),
    "hierarchy_warning": (C.c_char_p, [vp, L]),
    "hierarchy_report": (I, [vp, f64p, f64p]),
    "hierarchy_setup_ms": (I, [vp, f64p]),
    "vcycle": (I, [vp, L, f64p, f64p]),
    "kcycle": (I, [vp, C.POINTER(CycleConfigC), L, f64p, f64p]),
    "apply_preconditioner": (I, [vp, C.POINTER(CycleConfigC), f64p, f64p]),
    "pcg": (I, [csrp, f64p, f64p, vp, C.POINTER(CycleConfigC), C.POINTER(SolverConfigC), f64p,
                C.POINTER(SolveReportC)]),
    "fgmres": (I, [csrp, f64p, f64p, vp, C.POINTER(CycleConfigC), C.POINTER(SolverConfigC), f64p,
                   C.POINTER(SolveReportC)]),
    "pcg_cb": (I, [csrp, f64p, f64p, PRECOND_FN, vp, C.POINTER(SolverConfigC), f64p,
                   C.POINTER(SolveReportC)]),
    "fgmres_cb": (I, [csrp, f64p, f64p, PRECOND_FN, vp, C.POINTER(SolverConfigC), f64p,
                      C.POINTER(SolveReportC)]),
    "setup_and_solve": (I, [csrp, f64p, f64p, f64p, C.POINTER(SetupConfigC),
                            C.POINTER(CycleConfigC), C.POINTER(SolverConfigC), f64p,
                            C.POINTER(SolveReportC)]),
    "generate_poisson": (I, [I, L, L, L, C.c_double, I, csrp]),
    "random_vector": (I, [L, C.c_uint64, f64p]),
    "generate_jump27": (I, [L, L, L, C.c_double, L, csrp]),
    "set_num_threads": (None, [I]),
    "num_threads": (I, []),
    # product-only entry points
    "version": (C.c_char_p, []),
    "init": (I, [I]),
    "synchronize": (I, []),
    "kernel_launches": (L, []),
    "dmatrix_from_host": (I, [csrp, C.POINTER(vp)]),
    "dmatrix_poisson": (I, [I, L, L, L, C.c_double, I, C.POINTER(vp)]),
    "dmatrix_jump27": (I, [L, L, L, C.c_double, L, C.POINTER(vp)]),
    "dmatrix_size": (I, [vp, i64p, i64p]),
    "dmatrix_format": (I, [vp, i32p]),
    "dmatrix_to_host": (I, [vp, csrp]),
    "dmatrix_free": (None, [vp]),
    "setup_hierarchy_device": (I, [vp, C.POINTER(SetupConfigC), C.POINTER(vp)]),
    "solve_device": (I, [vp, C.POINTER(CycleConfigC), C.POINTER(SolverConfigC), f64p,
                         C.POINTER(SolveReportC)]),
    "profile_enable": (I, [I]),
    "profile_read": (I, [I, f64p, i64p, f64p]),
    "bench_spmv": (I, [vp, I, f64p, f64p]),
    "bench_dot": (I, [L, I, I, I, f64p]),
    "bench_kernel": (I, [vp, I, I, f64p, f64p]),
    "hierarchy_level_dmatrix": (I, [vp, L, I, C.POINTER(vp)]),
    "set_exact_reductions": (None, [I]),
    "exact_reductions": (I, []),
    "set_value_dictionary": (None, [I]),
    "set_row_patterns": (None, [I]),
    "timer_start": (I, []),
    "timer_stop": (I, [f64p]),
    "setup_config_default": (None, [C.POINTER(SetupConfigC)]),
    # row-partitioned multi-GPU path
    "comm_nccl_unique_id": (I, [C.c_char_p]),
    "comm_init_nccl": (I, [I, I, C.c_char_p, C.POINTER(vp)]),
    "comm_run_threads": (I, [I, i32p, vp, vp]),
    "comm_barrier": (I, [vp]),
    "comm_rank": (I, [vp]),
    "comm_size": (I, [vp]),
    "comm_kind": (C.c_char_p, [vp]),
    "comm_free": (None, [vp]),
    "read_matrix_market_file": (I, [C.c_char_p, I, csrp]),
    "read_matrix_market": (I, [C.c_char_p, L, I, csrp]),
    "write_matrix_market_file": (I, [C.c_char_p, csrp]),
    "read_vector_market_file": (I, [C.c_char_p, f64p, L, i64p]),
    "write_vector_market_file": (I, [C.c_char_p, f64p, L]),
    "generate_poisson_rows": (I, [I, L, L, L, C.c_double, I, L, L, csrp]),
    "generate_jump27_rows": (I, [L, L, L, C.c_double, L, L, L, csrp]),
    "dist_matrix_from_host": (I, [vp, L, L, csrp, C.POINTER(vp)]),
    "dist_matrix_poisson": (I, [vp, I, L, L, L, C.c_double, I, C.POINTER(vp)]),
    "dist_matrix_jump27": (I, [vp, L, L, L, C.c_double, L, C.POINTER(vp)]),
    "dist_matrix_info": (I, [vp, i64p, i64p, i64p, i64p]),
    "dist_matrix_format": (I, [vp, C.POINTER(C.c_int32)]),
    "dist_matrix_free": (None, [vp]),
    "dist_setup": (I, [vp, vp, f64p, C.POINTER(SetupConfigC), L, C.POINTER(vp)]),
    "dist_solve": (I, [vp, C.POINTER(CycleConfigC), C.POINTER(SolverConfigC), f64p, f64p,
                       C.POINTER(SolveReportC)]),
    "dist_refresh_values": (I, [vp, f64p, L]),
    "dist_apply_preconditioner": (I, [vp, C.POINTER(CycleConfigC), f64p, f64p]),
    "dist_hierarchy_info": (I, [vp, i64p, i64p, f64p]),
    "dist_hierarchy_level_size": (I, [vp, L, i64p, i64p]),
    "dist_hierarchy_level_A": (I, [vp, L, csrp]),
    "dist_hierarchy_level_transfer": (I, [vp, L, i64p, f64p, i32p]),
    "dist_hierarchy_level_B": (I, [vp, L, f64p]),
    "dist_hierarchy_level_omega": (I, [vp, L, f64p]),
    "dist_hierarchy_n_warnings": (L, [vp]),
    "dist_hierarchy_warning": (C.c_char_p, [vp, L]),
    "dist_hierarchy_free": (None, [vp]),
    "cycle_config_default": (None, [C.POINTER(CycleConfigC)]),
    "solver_config_default": (None, [C.POINTER(SolverConfigC)]),
}

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# AGGMG_LIB: an alternative build of the product library (kernel-variant experiments)
PRODUCT_LIB = os.environ.get("AGGMG_LIB") or os.path.join(REPO, "paper_1403_1649_b200", "lib",
                                                          "libaggmg_b200.so")


class LibraryMissing(RuntimeError):
    pass


class Lib:
    """A loaded implementation of the interface: fn(name) returns the bound symbol."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise LibraryMissing(f"{path} is not built (run __graft_entry__.build() or `make`)")
        self.path = path
        self.prefix = prefix
        self.cdll = C.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        self._cache = {}

    def has(self, name: str) -> bool:
        try:
            getattr(self.cdll, self.prefix + name)
            return True
        except AttributeError:
            return False

    def fn(self, name: str):
        f = self._cache.get(name)
        if f is None:
            f = getattr(self.cdll, self.prefix + name)
            res, args = SIGNATURES[name]
            f.restype = res
            f.argtypes = args
            self._cache[name] = f
        return f
