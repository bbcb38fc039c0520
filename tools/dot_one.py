#!/usr/bin/env python
"""One reference-order (chunked) dot product of n elements (ncu target)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1403_1649_b200 import aggmg as M  # noqa: E402

lib = M.b200().lib
assert lib.fn("init")(0) == 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 143921
ms = C.c_double()
assert lib.fn("bench_dot")(n, 1, 1, 2, C.byref(ms)) == 0
print(f"n={n}: {ms.value * 1e3:.1f} us")
