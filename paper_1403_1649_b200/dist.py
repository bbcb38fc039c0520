"""Row-partitioned (multi-GPU) AMG: Python face of the aggmg_comm_* / aggmg_dist_* C-ABI.

One rank per GPU.  The same rank code runs either

  * under torchrun, one process per GPU, over NCCL (``nccl_comm``), or
  * as R threads of one process (``run_threads``), each with its own CUDA stream and
    device (devices may repeat) — how the partitioned path is exercised on one B200.

Every method of DistMatrix / DistHierarchy is collective: all ranks call it in the same
order.  Level exports (``level_A`` ...) gather onto rank 0; other ranks receive ``None``.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Callable, List, Optional

import numpy as np

from . import _abi
from .aggmg import (CSR, CudaError, Error, SetupConfig, CycleConfig, SolverConfig, SolveReport,
                    SolveResult, SparseMatrix, b200, _f64, _p)


def _lib():
    return b200().lib


def _check(rc: int):
    if rc != 0:
        msg = _lib().fn("last_error")().decode()
        raise (CudaError if rc == 2 else Error)(msg)


class Comm:
    def __init__(self, handle, owned: bool):
        self._h = handle
        self._owned = owned

    @property
    def rank(self) -> int:
        return _lib().fn("comm_rank")(self._h)

    @property
    def size(self) -> int:
        return _lib().fn("comm_size")(self._h)

    @property
    def kind(self) -> str:
        return _lib().fn("comm_kind")(self._h).decode()

    def barrier(self):
        _check(_lib().fn("comm_barrier")(self._h))

    def close(self):
        if self._owned and self._h:
            _lib().fn("comm_free")(self._h)
        self._h = None


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().fn("comm_nccl_unique_id")(buf))
    return buf.raw


def nccl_comm(rank: int, size: int, uid: bytes, device: int) -> Comm:
    """One process per GPU: call on every rank with the id rank 0 created."""
    _check(_lib().fn("init")(device))
    h = C.c_void_p()
    _check(_lib().fn("comm_init_nccl")(rank, size, C.c_char_p(uid), C.byref(h)))
    return Comm(h, owned=True)


def run_threads(nranks: int, fn: Callable[[Comm, int], None],
                devices: Optional[List[int]] = None) -> None:
    """Run fn(comm, rank) on nranks rank threads of this process (in-process transport)."""
    errors = {}
    lock = threading.Lock()

    def tramp(hcomm, rank, _user):
        try:
            fn(Comm(hcomm, owned=False), rank)
            return 0
        except BaseException as e:  # noqa: BLE001 - reported through the runner
            with lock:
                errors[rank] = e
            return 1

    cb = _abi.RANK_FN(tramp)
    devs = (C.c_int32 * nranks)(*(devices or [0] * nranks))
    rc = _lib().fn("comm_run_threads")(nranks, devs, C.cast(cb, C.c_void_p), None)
    if errors:
        first = errors[min(errors)]
        # a rank that failed on its own is the root cause; others were woken by the abort
        for r in sorted(errors):
            if "aborted" not in str(errors[r]):
                first = errors[r]
                break
        raise first
    _check(rc)


def host_rows(kind: str, row0: int, nrows: int, nx: int, ny: int, nz: int = 1,
              epsilon: float = 1.0, dims: int = 3, jump: float = 1e6, block: int = 32) -> SparseMatrix:
    """Host slab [row0, row0 + nrows) of a generator matrix (global column ids)."""
    b = b200()
    if kind == "jump27":
        return b._csr_out("generate_jump27_rows", nx, ny, nz, jump, block, row0, nrows)
    return b._csr_out("generate_poisson_rows", dims, nx, ny, nz, epsilon, -1, row0, nrows)


class DistMatrix:
    def __init__(self, comm: Comm, handle):
        self.comm = comm
        self._h = handle

    @staticmethod
    def from_rows(comm: Comm, n_global: int, row0: int, rows: SparseMatrix) -> "DistMatrix":
        h = C.c_void_p()
        c = rows._c()
        _check(_lib().fn("dist_matrix_from_host")(comm._h, n_global, row0, C.byref(c), C.byref(h)))
        return DistMatrix(comm, h)

    @staticmethod
    def from_global(comm: Comm, A: SparseMatrix, part: Optional[List[int]] = None) -> "DistMatrix":
        """Slice this rank's rows out of a global host matrix (even partition by default)."""
        n, P, r = A.n_rows, comm.size, comm.rank
        part = part or [n * q // P for q in range(P + 1)]
        r0, r1 = part[r], part[r + 1]
        ro = A.row_offsets[r0:r1 + 1] - A.row_offsets[r0]
        lo, hi = A.row_offsets[r0], A.row_offsets[r1]
        rows = SparseMatrix(r1 - r0, A.n_cols, ro.copy(), A.col_indices[lo:hi].copy(),
                            A.values[lo:hi].copy())
        return DistMatrix.from_rows(comm, n, r0, rows)

    @staticmethod
    def poisson(comm: Comm, dims: int, nx: int, ny: int, nz: int = 1, epsilon: float = 1.0,
                weak_axis: int = -1) -> "DistMatrix":
        h = C.c_void_p()
        _check(_lib().fn("dist_matrix_poisson")(comm._h, dims, nx, ny, nz, epsilon, weak_axis,
                                                 C.byref(h)))
        return DistMatrix(comm, h)

    @staticmethod
    def jump27(comm: Comm, nx: int, ny: int, nz: int, jump: float = 1e6, block: int = 32):
        h = C.c_void_p()
        _check(_lib().fn("dist_matrix_jump27")(comm._h, nx, ny, nz, jump, block, C.byref(h)))
        return DistMatrix(comm, h)

    def info(self):
        v = [C.c_int64() for _ in range(4)]
        _check(_lib().fn("dist_matrix_info")(self._h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)  # n_global, row0, n_local, nnz_local

    def free(self):
        if self._h:
            _lib().fn("dist_matrix_free")(self._h)
        self._h = None


class DistHierarchy:
    def __init__(self, comm: Comm, handle):
        self.comm = comm
        self._h = handle

    def info(self):
        nl, nd, ms = C.c_int64(), C.c_int64(), C.c_double()
        _check(_lib().fn("dist_hierarchy_info")(self._h, C.byref(nl), C.byref(nd), C.byref(ms)))
        return nl.value, nd.value, ms.value  # total levels, distributed levels, setup ms

    def n_levels(self) -> int:
        return self.info()[0]

    def level_size(self, k: int):
        n, nnz = C.c_int64(), C.c_int64()
        _check(_lib().fn("dist_hierarchy_level_size")(self._h, k, C.byref(n), C.byref(nnz)))
        return n.value, nnz.value

    def level_A(self, k: int) -> Optional[SparseMatrix]:
        out = CSR()
        _check(_lib().fn("dist_hierarchy_level_A")(self._h, k, C.byref(out)))
        if self.comm.rank != 0:
            return None
        try:
            n, nnz = out.n_rows, out.nnz
            ro = np.ctypeslib.as_array(out.row_offsets, shape=(n + 1,)).copy()
            ci = np.ctypeslib.as_array(out.col_indices, shape=(max(nnz, 1),))[:nnz].copy()
            va = np.ctypeslib.as_array(out.values, shape=(max(nnz, 1),))[:nnz].copy()
        finally:
            _lib().fn("csr_free")(C.byref(out))
        return SparseMatrix(out.n_rows, out.n_cols, ro, ci, va)

    def level_transfer(self, k: int):
        n = self.level_size(k)[0]
        a = np.zeros(n, dtype=np.int64)
        p = np.zeros(n)
        sw = C.c_int32()
        _check(_lib().fn("dist_hierarchy_level_transfer")(self._h, k, _p(a, _abi.i64p),
                                                           _p(p, _abi.f64p), C.byref(sw)))
        return (a, p, sw.value) if self.comm.rank == 0 else None

    def level_B(self, k: int):
        B = np.zeros(self.level_size(k)[0])
        _check(_lib().fn("dist_hierarchy_level_B")(self._h, k, _p(B, _abi.f64p)))
        return B if self.comm.rank == 0 else None

    def level_omega(self, k: int):
        w = C.c_double(0.0)
        _check(_lib().fn("dist_hierarchy_level_omega")(self._h, k, C.byref(w)))
        return w.value

    def warnings(self) -> List[str]:
        f, g = _lib().fn("dist_hierarchy_n_warnings"), _lib().fn("dist_hierarchy_warning")
        return [g(self._h, i).decode() for i in range(f(self._h))]

    def solve(self, solver: Optional[SolverConfig] = None, cycle: Optional[CycleConfig] = None,
              b_local=None, n_local: Optional[int] = None) -> SolveResult:
        solver, cycle = solver or SolverConfig(), cycle or CycleConfig()
        hist = np.zeros(solver.max_iters + 2)
        rep = _abi.SolveReportC()
        rep.history = _p(hist, _abi.f64p)
        rep.history_capacity = hist.shape[0]
        x = np.zeros(n_local) if n_local is not None else None
        bp = _p(_f64(b_local), _abi.f64p) if b_local is not None else None
        cc, sc = cycle._c(), solver._c()
        _check(_lib().fn("dist_solve")(self._h, C.byref(cc), C.byref(sc), bp,
                                       _p(x, _abi.f64p) if x is not None else None, C.byref(rep)))
        return SolveResult(x, SolveReport(bool(rep.converged), rep.iterations,
                                          hist[: rep.history_length].tolist(), 0.0,
                                          rep.solve_seconds, rep.note.decode()))

    def refresh_values(self, new_values_local) -> None:
        """refresh_values (hierarchy.hpp:64): new values of this rank's level-0 rows."""
        v = _f64(new_values_local)
        _check(_lib().fn("dist_refresh_values")(self._h, _p(v, _abi.f64p), v.shape[0]))

    def apply_preconditioner(self, r_local, cycle: Optional[CycleConfig] = None) -> np.ndarray:
        r = _f64(r_local)
        z = np.zeros_like(r)
        cc = (cycle or CycleConfig())._c()
        _check(_lib().fn("dist_apply_preconditioner")(self._h, C.byref(cc), _p(r, _abi.f64p),
                                                       _p(z, _abi.f64p)))
        return z

    def free(self):
        if self._h:
            _lib().fn("dist_hierarchy_free")(self._h)
        self._h = None


def setup(comm: Comm, A: DistMatrix, config: Optional[SetupConfig] = None, B0_local=None,
          agglomerate_rows: int = 0) -> DistHierarchy:
    config = config or SetupConfig()
    h = C.c_void_p()
    cfg = config._c()
    Bp = _p(_f64(B0_local), _abi.f64p) if B0_local is not None else None
    _check(_lib().fn("dist_setup")(comm._h, A._h, Bp, C.byref(cfg), agglomerate_rows, C.byref(h)))
    return DistHierarchy(comm, h)
