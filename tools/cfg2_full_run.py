"""cfg2 full run (t_end = 48) -- one-off long-run parity check (dev tool).
    python tools/cfg2_full_run.py oracle LAM out.npz      # CPU oracle (slow)
    python tools/cfg2_full_run.py gpu LAM out.npz         # libhsgn on cuda:0
    python tools/cfg2_full_run.py compare a.npz b.npz
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import workloads as W  # noqa: E402


def main():
    mode = sys.argv[1]
    if mode == "compare":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        g = 9.81
        hm = np.max(np.abs(a["h"]))
        S = [hm, max(np.max(np.abs(a["q"])), np.sqrt(g * hm) * hm), np.max(np.abs(a["K"])),
             max(np.max(np.abs(a["W"])), float(a["lam"]) * float(a["dt"]))]
        errs = [np.max(np.abs(a[k] - b[k])) / s for k, s in zip("hqKW", S)]
        print("t", float(a["t"]), float(b["t"]), "steps", int(a["steps"]), int(b["steps"]),
              "scaled errors h q K W", ["%.2e" % e for e in errs])
        return
    lam, out = float(sys.argv[2]), sys.argv[3]
    nsteps = int(sys.argv[4]) if len(sys.argv) > 4 else None     # else run to t_end
    w = W.cfg2(lam)
    t0 = time.time()
    if mode == "oracle":
        from oracle import oracle as O
        o = O.Oracle(w.n, w.dx, lam=lam, bc=w.bc, filter_sigma=w.filter_sigma)
        if nsteps:
            U, t, steps, _ = o.run(w.state(0), cfl=w.cfl, mcfl=w.mcfl, steps=nsteps)
        else:
            U, t, steps, _ = o.run(w.state(0), cfl=w.cfl, mcfl=w.mcfl, t_end=w.t_end)
        dt = o.dt(U, w.cfl, w.mcfl)[0]
    else:
        from paper_2510_07539_b200 import hsgn
        s = hsgn.solver_for(w)
        if nsteps:
            s.run_steps(nsteps)
        else:
            s.advance_to(w.t_end)
        (h, q, K, Wf), tt = s.get_state(device=False)
        U, t = [h[0], q[0], K[0], Wf[0]], float(tt[0])
        dt = 0.0
        steps = s.diagnostics()["steps"]
    np.savez(out, h=U[0], q=U[1], K=U[2], W=U[3], t=t, steps=steps, lam=lam, dt=dt)
    print(mode, "lam", lam, "steps", steps, "t", t, "wall %.1f s" % (time.time() - t0))


if __name__ == "__main__":
    main()
