"""Per-field / per-step parity probe (dev tool, needs a GPU):
    python tools/parity_probe.py cfg5 20   |   python tools/parity_probe.py cfg2 14
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as O  # noqa: E402
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402

which, lg = sys.argv[1], int(sys.argv[2])
cases = []
if which == "cfg5":
    cases.append(W.cfg5_workload(1 << lg))
elif which == "cfg2":
    for lam in (100.0, 1e4):
        cases.append(W.cfg2(lam, n=1 << lg))
for w in cases:
    s = hsgn.solver_for(w)
    o = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc, b=w.b, filter_sigma=w.filter_sigma)
    U = w.state(0)
    done = 0
    for k in (1, 1, 3, 5):
        s.run_steps(k)
        U, *_ = o.run(U, cfl=w.cfl, mcfl=w.mcfl, steps=k)
        done += k
        (h, q, K, Wf), t = s.get_state(device=False)
        errs = []
        for name, a, b in zip("hqKW", (h[0], q[0], K[0], Wf[0]), U):
            i = int(np.argmax(np.abs(a - b)))
            errs.append(f"{name}: {np.max(np.abs(a - b)) / np.max(np.abs(b)):.2e} @ {i} (|f|max {np.max(np.abs(b)):.3g})")
        print(w.name, "lam", w.lam[0], "steps", done, " | ".join(errs), "rho_max",
              s.diagnostics()["rho_max"], flush=True)
