"""Dev probe: cfg3-shaped ensemble, K timed SI steps (one graph with event
nodes) on the overlapped tiles (mode 0), cluster kernels (1), auto (2), tile-level
SPIKE (3) or member-resident (4); prints per-stage device ms and fractions of
the HBM roofline.  Usage: python tools/cl_probe.py [members] [steps] [mode] [cells] [cfl_imex]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07539_b200 import hsgn as hs          # noqa: E402
from paper_2510_07539_b200 import workloads as W      # noqa: E402

members = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cl = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cells = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
cfl = float(sys.argv[5]) if len(sys.argv) > 5 else None      # CFL_IMEX override (0: MCFL-only stepping)
w = W.cfg3(members=members, n=cells)
s = hs.solver_for(w)
if cfl is not None:
    s.set_params(w.g, w.lam, cfl, w.mcfl)
if cl == 4:                                   # member-resident stepping
    s.set_cluster(1)
    s.run_resident(3)
    ms = s.run_resident(steps)
    N = cells * members
    print(f"resident: {ms / steps * 1e3:.1f} us/step, rho_max {s.diagnostics()['rho_max']:.3g}, {2 * N * steps / (ms * 1e-3) / 1e9:.2f} G cell-stage/s")
    raise SystemExit
s.set_cluster(cl)
print("cluster", s.cluster, "spike", s.spike, "geometry", s.geometry, "cfl", cfl)
s.run_steps(3)
s.sync()
ms1, ms2, tot = s.run_steps_timed(steps, total=True)
N = cells * members
peak = 6536.7e9
t1, t2 = ms1 / steps * 1e-3, ms2 / steps * 1e-3
print(f"stage1 {t1*1e6:.1f} us ({64*N/t1/peak:.3f}), stage2 {t2*1e6:.1f} us ({96*N/t2/peak:.3f}), "
      f"step {tot/steps*1e3:.1f} us, {2*N*steps/(tot*1e-3)/1e9:.2f} G cell-stage/s, "
      f"rho_max {s.diagnostics()['rho_max']:.3g}")
