"""Rounding floor of the parity metric (reading A17): the oracle against the SAME
oracle source built with FMA contraction (oracle.Oracle(variant="fma")), on the
configs' own inputs.  Any two correct fp64 implementations of the scheme may
differ by about this much; the GPU parity bars are set from it
(tests/test_gpu_parity.py, A17).

For each case and checkpoint it reports, per field, the plain normwise
difference max_i |a - b| / max_i |b| and the scaled form of A17
(S_q = max(max|q|, sqrt(g h_max) h_max), S_W = max(max|W|, lam dt)).

    python tools/a17_floor.py [--quick] > profiles/r02_a17_floor.json
"""
import json
import math
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O                      # noqa: E402
from paper_2510_07539_b200 import workloads as W    # noqa: E402

QUICK = "--quick" in sys.argv


def metrics(a, b, lam, dt, g=9.81):
    hm = np.max(np.abs(b[0]))
    S = [hm, max(np.max(np.abs(b[1])), math.sqrt(g * hm) * hm), np.max(np.abs(b[2])),
         max(np.max(np.abs(b[3])), lam * dt)]
    plain = [float(np.max(np.abs(x - y)) / max(np.max(np.abs(y)), 1e-300)) for x, y in zip(a, b)]
    scaled = [float(np.max(np.abs(x - y)) / s) for x, y, s in zip(a, b, S)]
    return plain, scaled


def run_pair(w, m, checkpoints):
    out = []
    U = {v: w.state(m) for v in ("plain", "fma")}
    done = 0
    mk = lambda v: O.Oracle(w.n, w.dx, g=w.g, lam=float(w.lam[m]), bc=w.bc, b=w.b,
                            filter_sigma=w.filter_sigma, relax=w.meta.get("relax"), variant=v)
    orc = {v: mk(v) for v in U}
    for c in checkpoints:
        with ThreadPoolExecutor(2) as ex:
            res = dict(zip(U, ex.map(lambda v: orc[v].run(U[v], cfl=w.cfl, mcfl=w.mcfl, steps=c - done),
                                     list(U))))
        for v in U:
            U[v] = res[v][0]
        done = c
        dt = orc["plain"].dt(U["plain"], w.cfl, w.mcfl)[0]
        p, s = metrics(U["fma"], U["plain"], float(w.lam[m]), dt, w.g)
        out.append(dict(steps=c, plain=p, scaled=s))
    return out


def main():
    rep = {"what": __doc__.strip().splitlines()[0], "fields": ["h", "q", "K", "W"], "cases": {}}
    # the variant must really round differently
    w = W.cfg3(members=1, n=4096)
    a = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), filter_sigma=0.25).step(w.state(0), 0.01)
    b = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), filter_sigma=0.25, variant="fma").step(w.state(0), 0.01)
    rep["variant_differs"] = bool(any(not np.array_equal(x, y) for x, y in zip(a, b)))
    # cfg3: members with low / mid / high lambda
    w = W.cfg3(members=64)
    order = np.argsort(w.lam)
    for m in ([order[0], order[32], order[-1]] if not QUICK else [order[-1]]):
        rep["cases"][f"cfg3_m{m}_lam{w.lam[m]:.0f}"] = run_pair(w, int(m), [1, 200] if not QUICK else [1, 20])
    # cfg5 recipe at 2^20 cells (oracle-sized), 1 and 100 steps
    w5 = W.cfg5_workload(n=1 << 20 if not QUICK else 1 << 16)
    rep["cases"][f"cfg5_n{w5.n}"] = run_pair(w5, 0, [1, 100] if not QUICK else [1, 10])
    # cfg2 (lambda = 100) along the run to t = 48
    if not QUICK:
        w2 = W.cfg2(100.0)
        rep["cases"]["cfg2_lam100"] = run_pair(w2, 0, [1, 200, 2000, 6000, 12000, 22000])
    json.dump(rep, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
