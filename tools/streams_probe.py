"""Dev probe: the cfg3 ensemble as 1-4 independent solvers on
separate streams, wall time of 54 steps each -- whether interleaving kernels of
several member groups fills the last-wave tails.
    python tools/streams_probe.py
"""
import sys, time
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import torch
from paper_2510_07539_b200 import hsgn, workloads as W
full = W.cfg3(members=4096)
def mk(w):
    s = hsgn.solver_for(w); s.run_steps(18); s.sync(); return s
for parts in (1, 2, 3, 4):
    ws = [full.subset(range(p * 4096 // parts, (p + 1) * 4096 // parts)) for p in range(parts)]
    ss = [mk(w) for w in ws]
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for s in ss: s.run_steps(54)
        for s in ss: s.sync()
        dt = time.perf_counter() - t0
    print(parts, f"{2 * 4096 * 4096 * 54 / dt / 1e9:.2f} G cell-stage/s ({dt*1e3:.1f} ms)")
    for s in ss: s.close()
