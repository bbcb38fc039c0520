"""Full-size parity pins: per-level digests of a hierarchy and its solve (shared by the pin
generator make_fullsize_pins.py, which runs the UNMODIFIED reference, and by
tests/test_gpu_fullsize_pins.py, which checks the B200 path against the pins).

A level digest is the SHA-256 of the level's arrays in a fixed layout: the operator A
(row offsets, column ids as int64, values as their IEEE bit patterns), P and R likewise, the
near-null-space vector B, the smoother's inverse diagonal, and omega / rho as exact hex
floats.  Two hierarchies with equal digests are bit-identical level by level."""
import hashlib

import numpy as np

# name -> (generator, dims, nx, ny, nz, epsilon / jump, alpha, method)
CONFIGS = {
    "c1": ("poisson", 2, 512, 512, 1, 1.0, 0.25, "pcg"),
    "c2": ("poisson", 3, 256, 256, 256, 1.0, 0.5, "pcg"),
    "c3": ("poisson", 3, 384, 384, 384, 1e-3, 0.5, "fgmres"),
    "c4": ("jump27", 3, 256, 256, 256, 1e6, 0.5, "pcg"),
    "c5": ("poisson", 3, 512, 512, 512, 1.0, 0.5, "pcg"),
}
JUMP_BLOCK = 32  # bench.py / DESIGN.md §7
TOL, MAX_ITERS, RESTART = 1e-8, 500, 30


def _h(*arrays):
    s = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        if a.dtype == np.float64:
            a = a.view(np.uint64)
        s.update(memoryview(a).cast("B"))
    return s.hexdigest()


def csr_digest(A):
    return _h(np.array([A.n_rows, A.n_cols], dtype=np.int64), A.row_offsets, A.col_indices,
              A.values)


def level_digest(h, k):
    """Digest of level k of a Hierarchy (any backend of the Python binding)."""
    lvl = h.levels[k]
    out = {"n": lvl.n, "nnz": lvl.nnz, "A": csr_digest(lvl.A), "B": _h(lvl.B)}
    if k < h.coarsest():
        out["P"] = csr_digest(lvl.P)
        out["R"] = csr_digest(lvl.R)
        s = lvl.smoother
        out["inv_diag"] = _h(s.inv_diag)
        out["omega"] = float(s.omega).hex()
        out["rho"] = float(s.rho_est).hex()
    return out


def vec_digest(x):
    return _h(np.asarray(x, dtype=np.float64))
