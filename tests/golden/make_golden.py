"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref, built from
/root/reference by `make -C oracle ref`).  Run in the build container:

    python tests/golden/make_golden.py

Each fixture is a small .npz of inputs and reference outputs; tests/test_oracle.py pins
the C restatement against them on CPU and tests/test_gpu_golden.py pins the B200 path.
The worked example is the reference's own Eq. 8 case (test_galerkin.cpp:22-51,
acceptance_main.cpp:143-186)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1403_1649_b200 import aggmg as M  # noqa: E402


def csr_dict(prefix, A):
    return {f"{prefix}_shape": np.array([A.n_rows, A.n_cols]), f"{prefix}_ro": A.row_offsets,
            f"{prefix}_ci": A.col_indices, f"{prefix}_v": A.values}


def worked_example():
    entries = [(0, 0), (0, 1), (0, 5), (1, 0), (1, 1), (1, 3), (1, 6), (2, 2), (2, 4), (2, 7),
               (3, 1), (3, 3), (3, 4), (3, 5), (3, 6), (4, 2), (4, 3), (4, 4), (4, 7), (5, 0),
               (5, 3), (5, 5), (6, 1), (6, 3), (6, 6), (7, 2), (7, 4), (7, 7)]
    rows = np.array([e[0] for e in entries])
    cols = np.array([e[1] for e in entries])
    vals = np.ldexp(1.0, np.arange(len(entries)))
    ro = np.zeros(9, dtype=np.int64)
    np.add.at(ro, rows + 1, 1)
    return M.SparseMatrix(8, 8, np.cumsum(ro), cols, vals)


def main():
    from oracle.checkers import ref

    r = ref()
    out = {}
    # 1. Eq. 8 worked example: cache order and exact grouped sums
    A = worked_example()
    a = np.array([1, 0, 2, 0, 2, 1, 0, 2], dtype=np.int64)
    agg = M.Aggregation(8, 3, a, np.array([1, 0, 2]))
    c = r.build_galerkin_cache(A, agg)
    P = M.SparseMatrix(8, 3, np.arange(9), a, np.ones(8))
    Ac = r.apply_galerkin_cache(c, A, P)
    np.savez(os.path.join(HERE, "worked_example.npz"), assignment=a, **csr_dict("A", A),
             **csr_dict("Ac", Ac), entry=c.entry, entry_row=c.entry_row,
             segment_offsets=c.segment_offsets, slot_of_csr=c.slot_of_csr)

    # 2. full hierarchies + solves on small Poisson problems (cache path)
    cases = {
        "poisson2d_32": (dict(dims=2, nx=32, ny=32, nz=1, epsilon=1.0), 0.25, M.PCG),
        "aniso2d_40x24": (dict(dims=2, nx=40, ny=24, nz=1, epsilon=0.01), 0.25, M.FGMRES),
        "poisson3d_12": (dict(dims=3, nx=12, ny=12, nz=12, epsilon=1.0), 0.5, M.PCG),
        "aniso3d_14": (dict(dims=3, nx=14, ny=14, nz=14, epsilon=1e-3), 0.5, M.FGMRES),
    }
    for name, (spec, alpha, method) in cases.items():
        A = r.generate_poisson(spec["dims"], spec["nx"], spec["ny"], spec["nz"], spec["epsilon"])
        cfg = M.SetupConfig(alpha=alpha, coarse_size_max=40, reuse_caches=True)
        h = r.setup_hierarchy(A, None, cfg)
        d = {"spec": np.array([spec["dims"], spec["nx"], spec["ny"], spec["nz"]]),
             "epsilon": np.array(spec["epsilon"]), "alpha": np.array(alpha),
             "n_levels": np.array(h.n_levels())}
        for k, lvl in enumerate(h.levels):
            d.update(csr_dict(f"A{k}", lvl.A))
            d[f"B{k}"] = lvl.B
            if k < h.coarsest():
                d.update(csr_dict(f"P{k}", lvl.P))
                d[f"omega{k}"] = np.array(lvl.smoother.omega)
        sc = M.SolverConfig(method=method, tol=1e-8, max_iters=300, restart=30)
        fn = r.pcg if method == M.PCG else r.fgmres
        res = fn(A, np.ones(A.n_rows), None, h, M.CycleConfig(), sc)
        d["method"] = np.array(method)
        d["history"] = np.array(res.report.residual_history)
        d["x"] = res.x
        np.savez(os.path.join(HERE, f"{name}.npz"), **d)

    # 3. MIS(2) on S of a seeded random-ish graph (a 2-D grid with diagonals cut)
    A = r.generate_poisson(2, 30, 17)
    Cm = r.classic_strength(A, 0.25)
    S = r.symmetrize_pattern(Cm)
    infl = r.influence_counts(Cm)
    states = {str(s): r.mis2(S, infl, s).state for s in (1, 42, 2**40 + 3)}
    np.savez(os.path.join(HERE, "mis2_grid.npz"), **csr_dict("S", S), influence=infl,
             **{f"state_{k}": v for k, v in states.items()})
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
