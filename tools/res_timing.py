"""Per-step phase clocks of the member-resident kernel, CTA 0 of member 0 (dev
tool; needs an HSGN_EXP_TIMING=1 build passed as HSGN_LIB):
    HSGN_LIB=<timing .so> python tools/res_timing.py [members] [cells] [steps]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402

members = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
w = W.cfg1() if (members == 1 and cells == 1000) else W.cfg3(members=members, n=cells)
s = hsgn.solver_for(w)
f = s.L.hsgn_cl_counters
f.restype = C.c_int
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 32)()
s.run_resident(5)
f(buf, 1)
ms = s.run_resident(steps)
f(buf, 1)
v = np.array(list(buf), dtype=np.float64).reshape(2, 16)
n = v[1, 15]
print(f"{n:.0f} steps timed, {ms / steps * 1e3:.2f} us per step (device)")
names = {0: ["phase 1", "assembly+PCR", "publish", "separator wait", "separator solve", "recovery+phase 3",
             "E2/R2 formed+sent", "E2/R2 halo wait"],
         1: ["phase 1", "assembly+PCR", "publish", "separator wait", "separator solve", "recovery+phase 3",
             "filter rows sent", "filter rows wait", "filter+relax+U sent", "dt maxima + dt", "U halo wait"]}
tot = (v[0, :8].sum() + v[1, :11].sum()) / n
print(f"clocks per step {tot:.0f} (+ loop top {v[0, 15] / n:.0f})")
for st in range(2):
    for k, nm in enumerate(names[st]):
        print(f"  stage {st + 1} {nm:22s} {v[st, k] / n:8.0f}  ({100 * v[st, k] / n / tot:4.1f}%)")
