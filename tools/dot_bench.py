#!/usr/bin/env python
"""Device dot-product throughput: tree order vs the reference's chunked order."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

lib = M.b200().lib
assert lib.fn("init")(0) == 0
for n in (16_777_216, 1_505_380, 143_921):
    for np_ in (1, 2):
        for exact in (0, 1):
            ms = C.c_double()
            assert lib.fn("bench_dot")(n, np_, exact, 20, C.byref(ms)) == 0, lib.fn("last_error")()
            byts = 8.0 * n * 2 * np_
            print(f"n={n} np={np_} {'chunked' if exact else 'tree'}: {ms.value*1e3:.1f} us, "
                  f"{byts / ms.value / 1e6:.0f} GB/s (vectors re-read per product)")
