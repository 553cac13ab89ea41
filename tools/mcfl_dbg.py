import sys; sys.path.insert(0, "/root/repo")
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import gpu_solver
from paper_2510_07539_b200 import hsgn as hs
for mode in (1, 3, 0):
    w = W.cfg3(members=1, first_member=144)
    w.cfl, w.mcfl = 0.0, 0.5
    s = gpu_solver(w)
    s.set_cluster(mode)
    print("mode", mode, s.cluster, s.spike, s.geometry)
    for k in range(25):
        try:
            s.run_steps(1); s.sync()
            d = s.diagnostics()
            print(k + 1, d["steps"], "%.4g" % d["rho_max"], "%.4g" % d["min_kappa"], "%.6g" % d["t_max"])
        except hs.HsgnError as e:
            print(k + 1, "ERR", e); break
