"""Dev probe: SPIKE across slabs (group transport) vs the single domain on SPIKE:
separators of aligned tiles (n = 24 x 512, 2 slabs of 12 tiles)."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2510_07539_b200 import workloads as W, hsgn as hs
bc = sys.argv[1] if len(sys.argv) > 1 else "periodic"
w = W.random_smooth(24 * 512, 1, seed=2, amp=0.08, bc=(bc, bc))
w.filter_sigma = 0.0
single = hs.solver_for(w)
single.set_cluster(3)
solvers, edges = hs.slab_solvers(w, 2, align=4)
for sv in solvers:
    sv.set_cluster(3)
g = hs.Group(solvers)
w.filter_sigma = 0.0
hs_ = hs
single.set_scheme("si", 1) if False else None
# one stage only: 1-stage tableau
tab = hs.euler_tableau()
single.set_tableau(tab)
for sv in solvers:
    sv.set_tableau(tab)
single.step()
g.run_steps(1)
L = single.debug_copy(0, 24)
tips = single.debug_copy(5, 24 * 12).reshape(24, 12)
for i, sv in enumerate(solvers):
    Ls = sv.debug_copy(0, 12)
    yvw = sv.debug_copy(1, 36).reshape(3, 12)
    elfr = sv.debug_copy(2, 2)
    nx = sv.debug_copy(3, 6)
    al = sv.debug_copy(4, 12).reshape(2, 6)
    t = sv.debug_copy(5, 12 * 12).reshape(12, 12)
    print("slab", i, "L diff", np.max(np.abs(Ls - L[12 * i:12 * i + 12])), "elfr", elfr,
          "exact El/Fr", L[(12 * i - 1) % 24], L[(12 * i + 12) % 24])
    print("   Y-L", np.abs(yvw[0] - L[12 * i:12 * i + 12]).max(), "V", np.abs(yvw[1]).max(), "W", np.abs(yvw[2]).max())
    print("   tips diff", np.abs(t - tips[12 * i:12 * i + 12]).max(axis=0))
    print("   nx", nx, "exact", tips[(12 * i + 12) % 24, 6:12])
    print("   all", al)
