import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2510_07539_b200 import workloads as W, hsgn as hs
from tests.test_gpu_parity import gpu_solver
for ln in [int(x) for x in (sys.argv[1:] or (20, 22, 24, 25, 26))]:
    w = W.cfg5_workload(1 << ln)
    a = gpu_solver(w); a.set_cluster(0)
    b = gpu_solver(w); b.set_cluster(3)
    a.step(); 
    try:
        b.step(); b.sync()
        (x, tx), (y, ty) = a.get_state(device=False), b.get_state(device=False)
        d = max(np.max(np.abs(x[k][0] - y[k][0])) / np.max(np.abs(x[k][0])) for k in range(4))
        print(ln, b.spike, "max rel diff %.2e" % d, flush=True)
    except Exception as e:
        print(ln, b.spike, "ERR", e, flush=True)
    del a, b
