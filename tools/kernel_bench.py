#!/usr/bin/env python
"""Per-kernel HBM throughput of the CSR-stream SpMV family on the c2 hierarchy
(3-D Poisson 256^3): level-0 operator, level-0 restriction R, level-1 operator.
Prints one JSON object; used for the roofline rows of DESIGN.md and under ncu for
profiles/ (ncu ... python tools/kernel_bench.py --reps 3)."""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1403_1649_b200 import aggmg as M  # noqa: E402

KINDS = {0: "spmv", 1: "residual", 2: "jacobi_zero+residual", 3: "jacobi", 4: "spmv+dot",
         5: "spmv*invdiag", 6: "jacobi+dot2", 7: "sgs"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kinds", default="0,1,2,3,4")
    ap.add_argument("--only", default="", help="e.g. L1.A:0 — run just this matrix:kind")
    ap.add_argument("--problem", default="c2", choices=["c1", "c2", "c4"],
                    help="c1: 5-point Poisson n^2; c2: 7-point Poisson n^3; "
                         "c4: 27-point jump 1e6 (32^3 blocks) n^3")
    args = ap.parse_args()
    lib = M.b200().lib
    assert lib.fn("init")(0) == 0, lib.fn("last_error")()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
    dm = C.c_void_p()
    if args.problem == "c4":
        assert lib.fn("dmatrix_jump27")(args.n, args.n, args.n, 1e6, 32, C.byref(dm)) == 0
    elif args.problem == "c1":
        assert lib.fn("dmatrix_poisson")(2, args.n, args.n, 1, 1.0, -1, C.byref(dm)) == 0
    else:
        assert lib.fn("dmatrix_poisson")(3, args.n, args.n, args.n, 1.0, -1, C.byref(dm)) == 0
    cfg = M.SetupConfig(alpha=0.25 if args.problem == "c1" else 0.5, reuse_caches=True)._c()
    h = C.c_void_p()
    assert lib.fn("setup_hierarchy_device")(dm, C.byref(cfg), C.byref(h)) == 0
    mats = {"L0.A": dm}
    for name, k, which in (("L0.R", 0, 1), ("L1.A", 1, 0), ("L1.R", 1, 1), ("L2.A", 2, 0)):
        m = C.c_void_p()
        assert lib.fn("hierarchy_level_dmatrix")(h, k, which, C.byref(m)) == 0
        mats[name] = m
    out = {}
    for name, m in mats.items():
        kinds = [int(k) for k in args.kinds.split(",")] if name.endswith(".A") else [0]
        if args.only:
            oname, okind = args.only.split(":")
            if oname != name:
                continue
            kinds = [int(okind)]
        for kind in kinds:
            ms, by = C.c_double(), C.c_double()
            rc = lib.fn("bench_kernel")(m, kind, args.reps, C.byref(ms), C.byref(by))
            assert rc == 0, lib.fn("last_error")()
            gbs = by.value / (ms.value / 1e3) / 1e9
            out[f"{name}:{KINDS[kind]}"] = {"avg_us": ms.value * 1e3, "bytes": by.value,
                                            "GBps": gbs, "frac_of_peak": gbs / peak}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
