"""Per-CTA phase clocks of the stage kernels (dev tool; needs an
HSGN_EXP_TIMING=1 build passed as HSGN_LIB):
    HSGN_LIB=.../variants/timing.so python tools/exp_timing.py [members]
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402

members = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = W.cfg3(members=members)
if "nofilter" in sys.argv[2:]:
    w.filter_sigma = 0.0
s = hsgn.solver_for(w)
L = s.L
f = L.hsgn_exp_counters
f.restype = C.c_int
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
s.run_steps(6)
s.sync()
f(buf, 1)
s.run_steps(18)
s.sync()
f(buf, 1)
v = np.array(list(buf), dtype=np.float64)
for k, name in ((0, "stage 1"), (8, "stage 2")):
    n = v[k + 3]
    a, b, c = v[k] / n, v[k + 1] / n, v[k + 2] / n
    tot = a + b + c
    print(f"{name}: CTAs {int(n)}  clocks/CTA: load wait {a:.0f} ({100*a/tot:.1f}%), "
          f"compute+store issue {b:.0f} ({100*b/tot:.1f}%), epilogue+drain {c:.0f} ({100*c/tot:.1f}%), total {tot:.0f}")
    p1, p2, p3 = v[k + 4] / n, v[k + 5] / n, v[k + 6] / n
    print(f"   compute split: in-place + phase 1 {p1:.0f}, phase 2 (assemble + solve) {p2:.0f}, "
          f"phase 3 + staging {p3:.0f}")
