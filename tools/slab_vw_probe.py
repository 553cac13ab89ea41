import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2510_07539_b200 import workloads as W, hsgn as hs
for bc in ("periodic", "wall"):
    w = W.random_smooth(512, 1, seed=5, amp=0.3, bc=(bc, bc))
    w.cfl, w.mcfl = 0.0, 0.3
    w.filter_sigma = 0.25
    solvers, _ = hs.slab_solvers(w, 8, align=4)
    for sv in solvers: sv.set_cluster(2)
    g = hs.Group(solvers)
    g.run_steps(1)
    print(bc, [np.abs(sv.debug_copy(1, 3)).round(14).tolist() for sv in solvers[:4]], solvers[0].diagnostics()["rho_max"])
