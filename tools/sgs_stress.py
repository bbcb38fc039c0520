#!/usr/bin/env python
"""Repeated level-scheduled SGS sweeps on every level of the 2-D 512^2 and 3-D 64^3 hierarchies,
bit-compared with the reference sweep each time (catches ordering races)."""
import sys, numpy as np
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
from paper_1403_1649_b200 import aggmg as M
from oracle import checkers  # noqa: E402
from helpers import bits
gpu = M.b200(); assert gpu.lib.fn("init")(0) == 0
ref = checkers.ref()
rng = np.random.default_rng(0)
for dim, nn, alpha in ((2, 512, 0.25), (3, 64, 0.5)):
    A0 = ref.generate_poisson(dim, nn, nn, nn if dim == 3 else 1)
    h = ref.setup_hierarchy(A0, None, M.SetupConfig(alpha=alpha, reuse_caches=True))
    for k, L in enumerate(h.levels[:4]):
        A = L.A
        s = ref.setup_smoother(A, M.JACOBI, 5, 0)
        st = M.SmootherState(M.SGS, s.inv_diag, 1.0, 1.0)
        b, x = rng.uniform(-1, 1, A.n_rows), rng.uniform(-1, 1, A.n_rows)
        want = bits(ref.smooth(st, A, b, x))
        bad = 0
        for rep in range(8):
            got = bits(gpu.smooth(st, A, b, x))
            nd = int(np.sum(got != want))
            bad += nd > 0
            if nd:
                idx = np.nonzero(got != want)[0]
                print(f"  dim{dim} L{k} rep{rep}: {nd} rows differ, first {idx[:5]}", flush=True)
        print(f"dim{dim} L{k} n={A.n_rows} bad_reps={bad}", flush=True)
