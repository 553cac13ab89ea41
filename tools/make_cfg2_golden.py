"""Writes tests/golden/cfg2_lam100_t48.npz: the ORACLE's state of the cfg2 dam
break (lambda = 100, 2^16 cells, walls, A19 filter) at t_end = 48, sampled
every 16th cell, and the rounding floor of the plain normwise metric at that
time (the same oracle source built with FMA contraction, reading A17): the
literal scheme's undular bore front amplifies round-off (A20), so two
fp64 implementations differ by a few percent there.  Calls only oracle/.

    python tools/make_cfg2_golden.py     (about 8 minutes: the two oracle builds in parallel)
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O                      # noqa: E402
from paper_2510_07539_b200 import workloads as W    # noqa: E402


def main():
    w = W.cfg2(100.0)

    def run(v):
        o = O.Oracle(w.n, w.dx, g=w.g, lam=100.0, bc=w.bc, filter_sigma=w.filter_sigma, variant=v)
        return o.run(w.state(0), cfl=w.cfl, mcfl=w.mcfl, t_end=w.t_end)

    with ThreadPoolExecutor(2) as ex:
        (U, t, st, mb), (Uf, tf, stf, _) = ex.map(run, ["plain", "fma"])
    floor = [float(np.max(np.abs(a - b)) / np.max(np.abs(b))) for a, b in zip(Uf, U)]
    out = os.path.join(ROOT, "tests", "golden", "cfg2_lam100_t48.npz")
    np.savez_compressed(out, sample=np.stack([f[::16] for f in U]), stride=16, t=t, steps=st,
                        steps_fma=stf, floor_plain=np.array(floor), min_beta=mb,
                        mass=np.sum(U[0]) * w.dx,
                        source="tools/make_cfg2_golden.py (oracle only): cfg2 lam 100, 2^16 cells, t_end 48")
    print(out, t, st, stf, floor)


if __name__ == "__main__":
    main()
