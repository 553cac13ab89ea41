"""Per-CTA phase clocks of the cluster stage kernels (dev tool; needs an
HSGN_EXP_TIMING=1 build passed as HSGN_LIB):
    python -c "from paper_2510_07539_b200 import build; build.build(out='paper_2510_07539_b200/lib/variants/timing.so', defines=['HSGN_EXP_TIMING=1'])"
    HSGN_LIB=paper_2510_07539_b200/lib/variants/timing.so python tools/cl_timing.py [members]
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402

members = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
w = W.cfg3(members=members)
s = hsgn.solver_for(w)
s.set_cluster(1)
f = s.L.hsgn_cl_counters
f.restype = C.c_int
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 32)()
s.run_steps(6)
s.sync()
f(buf, 1)
s.run_steps(18)
s.sync()
f(buf, 1)
v = np.array(list(buf), dtype=np.float64).reshape(2, 16)
names = ["load+E+barrier", "-", "-", "phase 1", "PCR", "publish+exchange", "sep.solve+recovery",
         "phase 3 (+filter)", "staging+store", "epilogue+drain"]
for st in range(2):
    n = v[st, 15]
    tot = v[st, :10].sum() / n
    print(f"stage {st + 1}: {n:.0f} CTAs, {tot:.0f} clocks per CTA")
    for k, nm in enumerate(names):
        print(f"   {nm:22s} {v[st, k] / n:8.0f}  ({100 * v[st, k] / n / tot:4.1f}%)")
