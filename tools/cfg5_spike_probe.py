"""Dev probe: cfg5 recipe at 2^ln cells -- a solver on the overlapped tiles (one
step, state read back on the device), then a fresh solver on tile-level SPIKE
in the memory it freed; variant 'zero' clears the second workspace first."""
import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2510_07539_b200 import workloads as W, hsgn as hs
ln = int(sys.argv[1]); variant = sys.argv[2] if len(sys.argv) > 2 else ""
n = 1 << ln


def run(mode, zero=False):
    (h, q, K, Wf, b), meta = W.cfg5(n, device="cuda")
    s = hs.Solver(n, 1, 0.0, meta["L"])
    if zero:
        s.workspace.zero_()
        torch.cuda.synchronize()
    s.set_params(9.81, meta["lam"], meta["cfl"], meta["mcfl"])
    s.set_bathymetry(b)
    s.set_filter(0.25)
    s.set_state(h, q, K, Wf)
    s.set_cluster(mode)
    try:
        dt = s.step(return_dt=True)[0]
        go, _ = s.get_state(device=True)
        print(mode, "dt", dt, "ok", float(go[0].max()), flush=True)
    except Exception as e:
        print(mode, "ERR", e, flush=True)


seq = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "3"])]
for i, mode in enumerate(seq):
    run(mode, zero=(variant == "zero" and i > 0))
