"""Python mirror of the reference ``aggmg`` C++ API (proj/core/include/aggmg/*.hpp).

Names, argument meaning, defaults and error behaviour follow the reference so parity
tests read like its own doctest suites.  Every call crosses the C-ABI
(include/aggmg_b200.h) into the product library:

    b200()    hand-written sm_100a kernels (fails loudly without a GPU build)

The CPU checkers the tests compare against (the C restatement and the unmodified
reference) live outside this package, in oracle/checkers.py (test infrastructure).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from ._abi import CSR, CycleConfigC, SetupConfigC, SolverConfigC, SolveReportC


class Error(RuntimeError):
    """aggmg::Error (reference error.hpp:14-17)."""


class CudaError(RuntimeError):
    """A CUDA failure inside the B200 library."""


# ---- value types -------------------------------------------------------------------


@dataclass
class SparseMatrix:
    """Canonical CSR (reference sparse.hpp:18-47)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    def at(self, i: int, j: int) -> float:
        lo, hi = self.row_offsets[i], self.row_offsets[i + 1]
        k = lo + np.searchsorted(self.col_indices[lo:hi], j)
        return float(self.values[k]) if k < hi and self.col_indices[k] == j else 0.0

    def to_dense(self) -> np.ndarray:
        D = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            lo, hi = self.row_offsets[i], self.row_offsets[i + 1]
            D[i, self.col_indices[lo:hi]] = self.values[lo:hi]
        return D

    @staticmethod
    def from_dense(D: np.ndarray) -> "SparseMatrix":
        rows, cols = np.nonzero(D)
        ro = np.zeros(D.shape[0] + 1, dtype=np.int64)
        np.add.at(ro, rows + 1, 1)
        return SparseMatrix(D.shape[0], D.shape[1], np.cumsum(ro), cols, D[rows, cols])

    def same_pattern(self, o: "SparseMatrix") -> bool:
        return (self.n_rows == o.n_rows and self.n_cols == o.n_cols
                and np.array_equal(self.row_offsets, o.row_offsets)
                and np.array_equal(self.col_indices, o.col_indices))

    def _c(self) -> CSR:
        c = CSR()
        c.n_rows, c.n_cols, c.nnz = self.n_rows, self.n_cols, self.nnz
        c.row_offsets = self.row_offsets.ctypes.data_as(_abi.i64p)
        c.col_indices = self.col_indices.ctypes.data_as(_abi.i64p)
        c.values = self.values.ctypes.data_as(_abi.f64p)
        return c


ZERO_DIAG_POSITIVE, ZERO_DIAG_FAIL = 0, 1
JACOBI, DAMPED_JACOBI, SGS = 0, 1, 2
CYCLE_V, CYCLE_K, CYCLE_HYBRID = 0, 1, 2
INNER_CG, INNER_GMRES = 0, 1
FGMRES, PCG = 0, 1


@dataclass
class SetupConfig:  # hierarchy.hpp:30-38
    alpha: float = 0.25
    coarse_size_max: int = 600
    max_levels: int = 25
    smoother: int = DAMPED_JACOBI
    arnoldi_m: int = 5
    seed: int = 42
    reuse_caches: bool = False

    def _c(self):
        c = SetupConfigC()
        c.alpha, c.coarse_size_max, c.max_levels = self.alpha, self.coarse_size_max, self.max_levels
        c.smoother, c.arnoldi_m, c.reuse_caches = self.smoother, self.arnoldi_m, int(self.reuse_caches)
        c.seed = self.seed
        return c


@dataclass
class CycleConfig:  # cycles.hpp:17-22
    kind: int = CYCLE_HYBRID
    k_levels: int = 2
    t: float = 0.25
    inner: int = INNER_GMRES

    def _c(self):
        c = CycleConfigC()
        c.kind, c.k_levels, c.t, c.inner = self.kind, self.k_levels, self.t, self.inner
        return c


@dataclass
class SolverConfig:  # krylov.hpp:16-21
    method: int = FGMRES
    tol: float = 1e-6
    max_iters: int = 200
    restart: int = 30

    def _c(self):
        c = SolverConfigC()
        c.method, c.tol, c.max_iters, c.restart = self.method, self.tol, self.max_iters, self.restart
        return c


@dataclass
class Mis2Result:  # aggregation.hpp:16-20
    state: np.ndarray
    roots: np.ndarray
    sweeps: int


@dataclass
class Aggregation:  # aggregation.hpp:32-37
    n_fine: int
    n_aggregates: int
    assignment: np.ndarray
    representatives: np.ndarray


@dataclass
class TransferOperators:  # transfer.hpp:14-18
    P: SparseMatrix
    R: SparseMatrix
    coarse_b: np.ndarray


@dataclass
class SmootherState:  # smoother.hpp:18-24
    kind: int
    inv_diag: np.ndarray
    omega: float
    rho_est: float


@dataclass
class SolveReport:  # krylov.hpp:23-30
    converged: bool
    iterations: int
    residual_history: List[float]
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0
    note: str = ""


@dataclass
class SolveResult:  # krylov.hpp:32-35
    x: np.ndarray
    report: SolveReport


@dataclass
class LevelStats:
    n: int
    nnz: int
    nnz_per_row: float


@dataclass
class HierarchyReport:  # hierarchy.hpp:66-76
    levels: List[LevelStats] = field(default_factory=list)
    grid_complexity: float = 0.0
    operator_complexity: float = 0.0


def _f64(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape[0] != n:
        raise Error("length mismatch")
    return a


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class GalerkinCache:
    """Handle to a GalerkinCache (galerkin.hpp:25-45); fields materialise on access."""

    def __init__(self, backend: "Backend", handle):
        self._b, self._h = backend, handle
        nf, nc, nnzf, nnzc = (C.c_int64() for _ in range(4))
        backend._call("galerkin_cache_info", self._h, C.byref(nf), C.byref(nc), C.byref(nnzf),
                      C.byref(nnzc))
        self.n_fine, self.n_coarse = nf.value, nc.value
        self._nnzf, self._nnzc = nnzf.value, nnzc.value
        arrs = {
            "coarse_row_offsets": self.n_coarse + 1, "coarse_col_indices": self._nnzc,
            "entry": self._nnzf, "entry_row": self._nnzf, "segment_offsets": self._nnzc + 1,
            "slot_of_csr": self._nnzf, "rows_by_coarse": self.n_fine,
            "agg_row_offsets": self.n_coarse + 1,
        }
        out = {k: np.zeros(max(v, 1), dtype=np.int64) for k, v in arrs.items()}
        backend._call("galerkin_cache_export", self._h,
                      *[_p(out[k], _abi.i64p) for k in arrs])
        for k, v in arrs.items():
            setattr(self, k, out[k][:v])

    def __del__(self):
        try:
            self._b.lib.fn("galerkin_cache_free")(self._h)
        except Exception:
            pass


class Level:
    """One level of a Hierarchy (hierarchy.hpp:21-28), materialised from the backend."""

    def __init__(self, h: "Hierarchy", k: int):
        self._h, self.k = h, k

    @property
    def A(self) -> SparseMatrix:
        return self._h._b._csr_out("hierarchy_level_A", self._h._h, self.k)

    @property
    def P(self) -> SparseMatrix:
        return self._h._b._csr_out("hierarchy_level_P", self._h._h, self.k)

    @property
    def R(self) -> SparseMatrix:
        return self._h._b._csr_out("hierarchy_level_R", self._h._h, self.k)

    @property
    def n(self) -> int:
        n, nnz = C.c_int64(), C.c_int64()
        self._h._b._call("hierarchy_level_size", self._h._h, self.k, C.byref(n), C.byref(nnz))
        return n.value

    @property
    def nnz(self) -> int:
        n, nnz = C.c_int64(), C.c_int64()
        self._h._b._call("hierarchy_level_size", self._h._h, self.k, C.byref(n), C.byref(nnz))
        return nnz.value

    @property
    def B(self) -> np.ndarray:
        out = np.zeros(self.n)
        self._h._b._call("hierarchy_level_B", self._h._h, self.k, _p(out, _abi.f64p))
        return out

    @property
    def smoother(self) -> SmootherState:
        om, rho = C.c_double(), C.c_double()
        inv = np.zeros(self.n)
        self._h._b._call("hierarchy_level_smoother", self._h._h, self.k, C.byref(om), C.byref(rho),
                         _p(inv, _abi.f64p))
        return SmootherState(self._h.config.smoother, inv, om.value, rho.value)

    def aggregation(self):
        """(assignment, n_aggregates, mis_sweeps) of the step k -> k+1 (B200 / oracle only)."""
        n = self.n
        a = np.zeros(n, dtype=np.int64)
        nc, sw = C.c_int64(), C.c_int32()
        self._h._b._call("hierarchy_level_aggregation", self._h._h, self.k, _p(a, _abi.i64p),
                         C.byref(nc), C.byref(sw))
        return a, nc.value, sw.value


class Hierarchy:
    """Hierarchy (hierarchy.hpp:40-48) held by one backend."""

    def __init__(self, backend: "Backend", handle, config: SetupConfig):
        self._b, self._h, self.config = backend, handle, config

    def __del__(self):
        try:
            if self._h:
                self._b.lib.fn("hierarchy_free")(self._h)
        except Exception:
            pass

    def n_levels(self) -> int:
        return int(self._b.lib.fn("hierarchy_n_levels")(self._h))

    def coarsest(self) -> int:
        return self.n_levels() - 1

    @property
    def levels(self) -> List[Level]:
        return [Level(self, k) for k in range(self.n_levels())]

    @property
    def warnings(self) -> List[str]:
        n = int(self._b.lib.fn("hierarchy_n_warnings")(self._h))
        return [self._b.lib.fn("hierarchy_warning")(self._h, i).decode() for i in range(n)]


class Backend:
    def __init__(self, lib: _abi.Lib, name: str):
        self.lib, self.name = lib, name

    # -- plumbing --
    def _call(self, name, *args):
        self._check(self.lib.fn(name)(*args))

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.fn("last_error")().decode()
            raise (CudaError if rc == 2 else Error)(msg)

    def _csr_out(self, name, *args) -> SparseMatrix:
        out = CSR()
        self._call(name, *args, C.byref(out))
        try:
            n, nnz = out.n_rows, out.nnz
            ro = np.ctypeslib.as_array(out.row_offsets, shape=(n + 1,)).copy()
            ci = np.ctypeslib.as_array(out.col_indices, shape=(max(nnz, 1),))[:nnz].copy()
            va = np.ctypeslib.as_array(out.values, shape=(max(nnz, 1),))[:nnz].copy()
        finally:
            self.lib.fn("csr_free")(C.byref(out))
        return SparseMatrix(out.n_rows, out.n_cols, ro, ci, va)

    # -- L1 (sparse.hpp / vector_ops.hpp) --
    def spmv(self, A: SparseMatrix, x) -> np.ndarray:
        x = _f64(x)
        if x.shape[0] != A.n_cols:
            raise Error(f"spmv: matrix has {A.n_cols} columns but vector has {x.shape[0]} entries")
        y = np.zeros(A.n_rows)
        c = A._c()
        self._call("spmv", C.byref(c), _p(x, _abi.f64p), _p(y, _abi.f64p))
        return y

    def transpose(self, A: SparseMatrix) -> SparseMatrix:
        c = A._c()
        return self._csr_out("transpose", C.byref(c))

    def dot(self, a, b) -> float:
        a, b = _f64(a), _f64(b)
        if a.shape != b.shape:
            raise Error("dot: length mismatch")
        out = C.c_double()
        self._call("dot", a.shape[0], _p(a, _abi.f64p), _p(b, _abi.f64p), C.byref(out))
        return out.value

    def norm2(self, a) -> float:
        a = _f64(a)
        out = C.c_double()
        self._call("norm2", a.shape[0], _p(a, _abi.f64p), C.byref(out))
        return out.value

    def axpy(self, a: float, x, y) -> np.ndarray:
        x, y = _f64(x), _f64(y).copy()
        if x.shape != y.shape:
            raise Error("axpy: length mismatch")
        self._call("axpy", x.shape[0], a, _p(x, _abi.f64p), _p(y, _abi.f64p))
        return y

    def scale(self, a: float, x) -> np.ndarray:
        x = _f64(x).copy()
        self._call("scale", x.shape[0], a, _p(x, _abi.f64p))
        return x

    # -- L2 setup components --
    def classic_strength(self, A: SparseMatrix, alpha: float, policy: int = ZERO_DIAG_POSITIVE):
        c = A._c()
        return self._csr_out("classic_strength", C.byref(c), alpha, policy)

    def influence_counts(self, Cm: SparseMatrix) -> np.ndarray:
        out = np.zeros(Cm.n_cols, dtype=np.int64)
        c = Cm._c()
        self._call("influence_counts", C.byref(c), _p(out, _abi.i64p))
        return out

    def symmetrize_pattern(self, Cm: SparseMatrix) -> SparseMatrix:
        c = Cm._c()
        return self._csr_out("symmetrize_pattern", C.byref(c))

    def mis2(self, S: SparseMatrix, influence, seed: int) -> Mis2Result:
        infl = np.ascontiguousarray(influence, dtype=np.int64)
        if infl.shape[0] != S.n_rows:
            raise Error("mis2: influence length mismatch")
        state = np.zeros(S.n_rows, dtype=np.int8)
        nr, sw = C.c_int64(), C.c_int32()
        c = S._c()
        self._call("mis2", C.byref(c), _p(infl, _abi.i64p), C.c_uint64(seed), _p(state, _abi.i8p),
                   C.byref(nr), C.byref(sw))
        return Mis2Result(state, np.nonzero(state == 1)[0].astype(np.int64), sw.value)

    def aggregate(self, S: SparseMatrix, A: SparseMatrix, mis: Mis2Result) -> Aggregation:
        n = S.n_rows
        state = np.ascontiguousarray(mis.state, dtype=np.int8)
        if state.shape[0] != n:
            raise Error("aggregate: state length mismatch")
        a = np.zeros(n, dtype=np.int64)
        reps = np.zeros(max(n, 1), dtype=np.int64)
        nc = C.c_int64()
        cs, ca = S._c(), A._c()
        self._call("aggregate", C.byref(cs), C.byref(ca), _p(state, _abi.i8p), _p(a, _abi.i64p),
                   _p(reps, _abi.i64p), C.byref(nc))
        return Aggregation(n, nc.value, a, reps[: nc.value].copy())

    def build_transfer(self, agg: Aggregation, fine_b) -> TransferOperators:
        b = _f64(fine_b)
        if b.shape[0] != agg.n_fine:
            raise Error("transfer: near-null-space vector length mismatch")
        a = np.ascontiguousarray(agg.assignment, dtype=np.int64)
        P, R = CSR(), CSR()
        cb = np.zeros(max(agg.n_aggregates, 1))
        self._call("build_transfer", agg.n_fine, agg.n_aggregates, _p(a, _abi.i64p),
                   _p(b, _abi.f64p), C.byref(P), C.byref(R), _p(cb, _abi.f64p))
        return TransferOperators(self._adopt(P), self._adopt(R), cb[: agg.n_aggregates].copy())

    def _adopt(self, out: CSR) -> SparseMatrix:
        try:
            n, nnz = out.n_rows, out.nnz
            ro = np.ctypeslib.as_array(out.row_offsets, shape=(n + 1,)).copy()
            ci = np.ctypeslib.as_array(out.col_indices, shape=(max(nnz, 1),))[:nnz].copy()
            va = np.ctypeslib.as_array(out.values, shape=(max(nnz, 1),))[:nnz].copy()
        finally:
            self.lib.fn("csr_free")(C.byref(out))
        return SparseMatrix(out.n_rows, out.n_cols, ro, ci, va)

    def galerkin_direct(self, R: SparseMatrix, A: SparseMatrix, P: SparseMatrix) -> SparseMatrix:
        cr, ca, cp = R._c(), A._c(), P._c()
        return self._csr_out("galerkin_direct", C.byref(cr), C.byref(ca), C.byref(cp))

    def build_galerkin_cache(self, A: SparseMatrix, agg: Aggregation) -> GalerkinCache:
        a = np.ascontiguousarray(agg.assignment, dtype=np.int64)
        h = C.c_void_p()
        c = A._c()
        self._call("build_galerkin_cache", C.byref(c), agg.n_aggregates, _p(a, _abi.i64p),
                   C.byref(h))
        return GalerkinCache(self, h)

    def apply_galerkin_cache(self, cache: GalerkinCache, A: SparseMatrix,
                             P: SparseMatrix) -> SparseMatrix:
        ca, cp = A._c(), P._c()
        return self._csr_out("apply_galerkin_cache", cache._h, C.byref(ca), C.byref(cp))

    def setup_smoother(self, A: SparseMatrix, kind: int = DAMPED_JACOBI, arnoldi_m: int = 5,
                       seed: int = 0) -> SmootherState:
        inv = np.zeros(A.n_rows)
        om, rho = C.c_double(), C.c_double()
        c = A._c()
        self._call("setup_smoother", C.byref(c), kind, arnoldi_m, C.c_uint64(seed),
                   _p(inv, _abi.f64p), C.byref(om), C.byref(rho))
        return SmootherState(kind, inv, om.value, rho.value)

    def smooth(self, s: SmootherState, A: SparseMatrix, b, x) -> np.ndarray:
        n = A.n_rows
        b, x = _f64(b), _f64(x).copy()
        if b.shape[0] != n or x.shape[0] != n:
            raise Error("smooth: vector length mismatch")
        inv = _f64(s.inv_diag)
        c = A._c()
        self._call("smooth", s.kind, _p(inv, _abi.f64p), s.omega, C.byref(c), _p(b, _abi.f64p),
                   _p(x, _abi.f64p))
        return x

    def hessenberg_eigenvalues(self, H: np.ndarray) -> np.ndarray:
        H = np.ascontiguousarray(H, dtype=np.float64)
        n = H.shape[0]
        re, im = np.zeros(n), np.zeros(n)
        self._call("hessenberg_eigenvalues", n, _p(H, _abi.f64p), _p(re, _abi.f64p),
                   _p(im, _abi.f64p))
        return re + 1j * im

    # -- L3 --
    def setup_hierarchy(self, A0: SparseMatrix, B0=None, config: Optional[SetupConfig] = None):
        config = config or SetupConfig()
        B = _f64(B0) if B0 is not None else np.ones(A0.n_rows)
        if B.shape[0] != A0.n_rows:
            raise Error("setup: near-null-space vector length mismatch")
        h = C.c_void_p()
        cfg = config._c()
        c = A0._c()
        self._call("setup_hierarchy", C.byref(c), _p(B, _abi.f64p), C.byref(cfg), C.byref(h))
        return Hierarchy(self, h, config)

    def refresh_values(self, h: Hierarchy, new_values) -> Hierarchy:
        v = _f64(new_values)
        self._call("refresh_values", h._h, _p(v, _abi.f64p), v.shape[0])
        return h

    def hierarchy_report(self, h: Hierarchy) -> HierarchyReport:
        r = HierarchyReport()
        sn = snnz = 0.0
        for lvl in h.levels:
            n, nnz = lvl.n, lvl.nnz
            r.levels.append(LevelStats(n, nnz, nnz / n if n else 0.0))
            sn += n
            snnz += nnz
        r.grid_complexity = sn / r.levels[0].n
        r.operator_complexity = snnz / r.levels[0].nnz
        return r

    # -- L4 cycles --
    def vcycle(self, h: Hierarchy, k: int, b, x) -> np.ndarray:
        b, x = _f64(b), _f64(x).copy()
        self._call("vcycle", h._h, k, _p(b, _abi.f64p), _p(x, _abi.f64p))
        return x

    def kcycle(self, h: Hierarchy, cfg: CycleConfig, k: int, b, x) -> np.ndarray:
        b, x = _f64(b), _f64(x).copy()
        c = cfg._c()
        self._call("kcycle", h._h, C.byref(c), k, _p(b, _abi.f64p), _p(x, _abi.f64p))
        return x

    def apply_preconditioner(self, h: Hierarchy, cfg: CycleConfig, r) -> np.ndarray:
        r = _f64(r)
        n = h.levels[0].n
        if r.shape[0] != n:
            raise Error("preconditioner: vector length mismatch")
        z = np.zeros(n)
        c = cfg._c()
        self._call("apply_preconditioner", h._h, C.byref(c), _p(r, _abi.f64p), _p(z, _abi.f64p))
        return z

    # -- L4 Krylov --
    def _krylov(self, name, A, b, x0, M, cycle, cfg):
        n = A.n_rows
        b = _f64(b)
        x0 = np.zeros(n) if x0 is None else _f64(x0)
        if b.shape[0] != n or x0.shape[0] != n:
            raise Error(f"{name}: vector length mismatch")
        cfg = cfg or SolverConfig()
        cycle = cycle or CycleConfig()
        x = np.zeros(n)
        hist = np.zeros(cfg.max_iters + 2)
        rep = SolveReportC()
        rep.history = _p(hist, _abi.f64p)
        rep.history_capacity = hist.shape[0]
        cc, sc, ca = cycle._c(), cfg._c(), A._c()
        if M is not None and not isinstance(M, Hierarchy):
            # any host callable r -> z (the reference's std::function Preconditioner)
            failure = []

            def thunk(r_ptr, z_ptr, nn, _user):
                try:
                    r = np.ctypeslib.as_array(r_ptr, shape=(nn,)).copy()
                    np.ctypeslib.as_array(z_ptr, shape=(nn,))[:] = _f64(M(r), nn)
                    return 0
                except Exception as e:  # noqa: BLE001 - re-raised after the C call
                    failure.append(e)
                    return 1

            cb = _abi.PRECOND_FN(thunk)
            rc = self.lib.fn(name + "_cb")(C.byref(ca), _p(b, _abi.f64p), _p(x0, _abi.f64p), cb,
                                           None, C.byref(sc), _p(x, _abi.f64p), C.byref(rep))
            if failure:
                raise failure[0]
            self._check(rc)
        else:
            self._call(name, C.byref(ca), _p(b, _abi.f64p), _p(x0, _abi.f64p),
                       M._h if M is not None else None, C.byref(cc), C.byref(sc),
                       _p(x, _abi.f64p), C.byref(rep))
        return SolveResult(x, SolveReport(bool(rep.converged), rep.iterations,
                                          hist[: rep.history_length].tolist(), 0.0,
                                          rep.solve_seconds, rep.note.decode()))

    def pcg(self, A, b, x0=None, M: Optional[Hierarchy] = None, cycle=None, cfg=None):
        return self._krylov("pcg", A, b, x0, M, cycle, cfg)

    def fgmres(self, A, b, x0=None, M: Optional[Hierarchy] = None, cycle=None, cfg=None):
        return self._krylov("fgmres", A, b, x0, M, cycle, cfg)

    def setup_and_solve(self, A: SparseMatrix, b, setup=None, cycle=None, solver=None, B0=None,
                        x0=None) -> SolveResult:
        n = A.n_rows
        setup, cycle, solver = setup or SetupConfig(), cycle or CycleConfig(), solver or SolverConfig()
        b = _f64(b, n)
        Bp = _p(_f64(B0, n), _abi.f64p) if B0 is not None else None
        xp = _p(_f64(x0, n), _abi.f64p) if x0 is not None else None
        x = np.zeros(n)
        hist = np.zeros(solver.max_iters + 2)
        rep = SolveReportC()
        rep.history = _p(hist, _abi.f64p)
        rep.history_capacity = hist.shape[0]
        ca, s1, s2, s3 = A._c(), setup._c(), cycle._c(), solver._c()
        self._call("setup_and_solve", C.byref(ca), _p(b, _abi.f64p), Bp, xp, C.byref(s1),
                   C.byref(s2), C.byref(s3), _p(x, _abi.f64p), C.byref(rep))
        return SolveResult(x, SolveReport(bool(rep.converged), rep.iterations,
                                          hist[: rep.history_length].tolist(), rep.setup_seconds,
                                          rep.solve_seconds, rep.note.decode()))

    # -- Matrix Market (matrix_market.hpp:23-35) --
    def read_matrix_market(self, path: str, allow_pattern: bool = False) -> SparseMatrix:
        return self._csr_out("read_matrix_market_file", str(path).encode(), int(allow_pattern))

    def read_matrix_market_text(self, text, allow_pattern: bool = False) -> SparseMatrix:
        data = text.encode() if isinstance(text, str) else bytes(text)
        return self._csr_out("read_matrix_market", data, len(data), int(allow_pattern))

    def write_matrix_market(self, path: str, A: SparseMatrix) -> None:
        ca = A._c()
        self._call("write_matrix_market_file", str(path).encode(), C.byref(ca))

    def read_vector_market(self, path: str) -> np.ndarray:
        n = C.c_int64()
        self._call("read_vector_market_file", str(path).encode(), None, 0, C.byref(n))
        x = np.zeros(n.value)
        self._call("read_vector_market_file", str(path).encode(), _p(x, _abi.f64p), n.value,
                   C.byref(n))
        return x

    def write_vector_market(self, path: str, x) -> None:
        x = _f64(x)
        self._call("write_vector_market_file", str(path).encode(), _p(x, _abi.f64p), x.shape[0])

    # -- inputs (poisson.hpp) --
    def generate_poisson(self, dims: int, nx: int, ny: int, nz: int = 1, epsilon: float = 1.0,
                         weak_axis: int = -1) -> SparseMatrix:
        return self._csr_out("generate_poisson", dims, nx, ny, nz, epsilon, weak_axis)

    def generate_jump27(self, nx: int, ny: int, nz: int, jump: float = 1e6,
                        block: int = 32) -> SparseMatrix:
        return self._csr_out("generate_jump27", nx, ny, nz, jump, block)


_product = None


def b200() -> Backend:
    """The product: the sm_100a kernels behind include/aggmg_b200.h."""
    global _product
    if _product is None:
        _product = Backend(_abi.Lib(_abi.PRODUCT_LIB, "aggmg_"), "b200")
    return _product


def ones_vector(n: int) -> np.ndarray:  # poisson.hpp:28
    return np.ones(n)
