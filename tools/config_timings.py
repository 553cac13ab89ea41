"""Time every BASELINE config on one GPU (dev tool; numbers for DESIGN.md section 9):
device time (CUDA events on the solver's stream) of the configured run and the
implied fp64 cell-stage updates/s.

    python tools/config_timings.py [cfg1 cfg2 cfg4 cfg5]
"""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2510_07539_b200 import hsgn  # noqa: E402
from paper_2510_07539_b200 import workloads as W  # noqa: E402


def timed(s, fn):
    st = s.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(st)
    out = fn()
    e1.record(st)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) / 1e3, time.perf_counter() - w0


def report(name, cells, steps, dev_s, wall_s, extra=""):
    rate = 2.0 * cells * steps / dev_s
    print(f"{name}: {steps} steps x {cells} cells: device {dev_s * 1e3:.1f} ms, wall {wall_s * 1e3:.1f} ms, "
          f"{rate / 1e9:.2f} G cell-stage/s {extra}", flush=True)


def main():
    which = sys.argv[1:] or ["cfg1", "cfg2", "cfg4", "cfg5"]
    torch.cuda.set_device(0)
    if "cfg1" in which:
        w = W.cfg1()
        s = hsgn.solver_for(w)
        s.advance_to(1.0)                       # warm-up (graph capture)
        s = hsgn.solver_for(w)
        _, dev, wall = timed(s, lambda: s.advance_to(w.t_end))
        report("cfg1 soliton to t_end = 20", w.n, s.diagnostics()["steps"], dev, wall)
    if "cfg2" in which:
        for lam in (1e2, 1e3, 1e4):
            w = W.cfg2(lam)
            s = hsgn.solver_for(w)
            _, dev, wall = timed(s, lambda: s.advance_to(w.t_end))
            report(f"cfg2 dam break lam {lam:g} to t_end = 48", w.n, s.diagnostics()["steps"], dev, wall)
    if "cfg4" in which:
        w = W.cfg4()
        s = hsgn.solver_for(w)
        s.run_steps(18)
        _, dev, wall = timed(s, lambda: s.run_steps(200))
        report("cfg4 bar, 4 lambdas x 2^20 cells, 200 steps", w.n * w.members, 200, dev, wall)
    if "cfg5" in which:
        (h, q, K, Wf, b), meta = W.cfg5(1 << 28, device="cuda")
        s = hsgn.Solver(1 << 28, 1, 0.0, meta["L"])
        s.set_params(9.81, meta["lam"], meta["cfl"], meta["mcfl"])
        s.set_bathymetry(b)
        s.set_filter(0.25)
        s.set_state(h, q, K, Wf)
        del h, q, K, Wf
        s.run_steps(6)
        _, dev, wall = timed(s, lambda: s.run_steps(100))
        report("cfg5 2^28 cells, 100 steps", 1 << 28, 100, dev, wall)


if __name__ == "__main__":
    main()
