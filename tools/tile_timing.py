"""Per-CTA phase clocks of the overlapped-tile stage kernels (dev tool; needs an
HSGN_EXP_TIMING=1 build passed as HSGN_LIB): python tools/tile_timing.py [members | cfg2]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "4096"
w = W.cfg2(1e2) if arg == "cfg2" else W.cfg3(members=int(arg))
s = hsgn.solver_for(w)
s.set_cluster(0)
f = s.L.hsgn_exp_counters
f.restype = C.c_int
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
s.run_steps(6)
s.sync()
f(buf, 1)
s.run_steps(18)
s.sync()
f(buf, 1)
v = np.array(list(buf), dtype=np.float64).reshape(2, 8)
names = ["load wait", "compute + store issue", "epilogue + drain", "-", "in-place + phase 1", "phase 2",
         "phase 3 + staging", "  of phase 2: PCR + recovery"]
for st in range(2):
    n = v[st, 3]
    tot = (v[st, 0] + v[st, 1] + v[st, 2]) / n
    print(f"stage {st + 1}: {n:.0f} CTAs, {tot:.0f} clocks per CTA")
    for k, nm in enumerate(names):
        if k != 3:
            print(f"   {nm:30s} {v[st, k] / n:8.0f}  ({100 * v[st, k] / n / tot:4.1f}%)")
