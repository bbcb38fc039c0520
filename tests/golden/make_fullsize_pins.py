"""Generate tests/golden/fullsize_pins.json from the UNMODIFIED reference (oracle/_ref) at the
BASELINE configurations' full sizes.  Test infrastructure; runs on a host with enough memory
and cores (the GPU box: 16 cores, 196 GB; c5's cache path needs ~90 GB), e.g.

    gpurun -- python tests/golden/make_fullsize_pins.py c2 c4 c3 c5

For each config: the reference's cache-path hierarchy (reuse_caches = true, the summation
order the B200 path reproduces) digested level by level (tests/golden/fullsize.py),
then the reference's PCG / FGMRES(30) with the hybrid K-cycle to 1e-8 from x0 = 0, b = ones:
iteration count, the full residual history (17 significant digits) and a digest of x.
The c4 matrix comes from the C restatement's 27-point generator (no reference generator
exists; the definition is DESIGN.md §7), passed to the reference as a host CSR."""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from fullsize import (CONFIGS, JUMP_BLOCK, MAX_ITERS, RESTART, TOL, csr_digest,  # noqa: E402
                      level_digest, vec_digest)
from oracle.checkers import oracle, ref  # noqa: E402
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

OUT = os.environ.get("PINS_OUT") or os.path.join(HERE, "fullsize_pins.json")


def run(name):
    gen, dims, nx, ny, nz, eps, alpha, method = CONFIGS[name]
    r = ref()
    threads = os.cpu_count() or 1
    r.lib.fn("set_num_threads")(threads)
    t0 = time.time()
    if gen == "jump27":
        A = oracle().generate_jump27(nx, ny, nz, eps, JUMP_BLOCK)
    else:
        A = r.generate_poisson(dims, nx, ny, nz, eps)
    cfg = M.SetupConfig(alpha=alpha, reuse_caches=True)
    t1 = time.time()
    h = r.setup_hierarchy(A, None, cfg)
    t2 = time.time()
    levels = [level_digest(h, k) for k in range(h.n_levels())]
    t3 = time.time()
    sc = M.SolverConfig(method=M.PCG if method == "pcg" else M.FGMRES, tol=TOL,
                        max_iters=MAX_ITERS, restart=RESTART)
    res = (r.pcg if method == "pcg" else r.fgmres)(A, np.ones(A.n_rows), None, h, M.CycleConfig(), sc)
    t4 = time.time()
    out = {
        "config": name, "generator": gen, "grid": [nx, ny, nz], "epsilon": eps, "alpha": alpha,
        "method": method, "n": A.n_rows, "nnz": A.nnz, "input": csr_digest(A),
        "levels": levels, "iterations": res.report.iterations,
        "converged": res.report.converged,
        "history": [float(v).hex() for v in res.report.residual_history],
        "x": vec_digest(res.x), "x_norm": float(np.linalg.norm(res.x)),
        "reference_seconds": {"generate": t1 - t0, "setup": t2 - t1, "digest": t3 - t2,
                              "solve": t4 - t3},
        "threads": threads,
    }
    print(f"{name}: {len(levels)} levels, {res.report.iterations} its, setup {t2 - t1:.1f} s, "
          f"solve {t4 - t3:.1f} s", flush=True)
    del h, A
    return out


def main(names):
    pins = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            pins = json.load(f)
    for name in names:
        pins[name] = run(name)
        with open(OUT, "w") as f:  # after every config: a later one may run out of time
            json.dump(pins, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
