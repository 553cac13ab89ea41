"""Dev probe: time per step of the cfg2 dam break (65536
cells, latency-bound) for the three kernel organisations and tile sizes.
    python tools/cfg2_modes.py
"""
import sys, time
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import torch
from paper_2510_07539_b200 import hsgn, workloads as W
for mode in ("default", "fused", "persistent"):
    for tc in (0, 256, 128):
        w = W.cfg2(100.0)
        kw = {"tile_cells": tc} if tc else {}
        s = hsgn.Solver(w.n, w.members, w.x_min, w.x_max, bc=w.bc, **kw)
        s.set_params(w.g, w.lam, w.cfl, w.mcfl)
        if w.filter_sigma > 0: s.set_filter(w.filter_sigma)
        if mode == "fused": s.set_fused(True)
        if mode == "persistent": s.set_persistent(True)
        s.set_state(w.h.reshape(-1), w.q.reshape(-1), w.K.reshape(-1), w.W.reshape(-1))
        s.run_steps(36); s.sync()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.run_steps(1800); s.sync()
        dt = time.perf_counter() - t0
        g = s.geometry
        print(mode, tc, "T", g.tile_cells, "tiles", g.tiles_per_member, "fused", s.fused, f"{dt/1800*1e6:.1f} us/step")
