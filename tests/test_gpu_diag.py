"""Boundary diagnostics (include/hsgn.h hsgn_diag): the coercivity monitor
min_kappa (kappa = beta of P:505-507 must stay > 0) and the
achieved Courant numbers of the next step, against the
oracle on the same inputs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import gpu_solver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cluster", [0, 1])
@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_min_kappa_matches_oracle(bc, cluster):
    w = W.random_smooth(2048, 3, seed=17, amp=0.1, bc=(bc, bc))
    s = gpu_solver(w)
    s.set_cluster(cluster)
    d0 = s.diagnostics()
    assert d0["min_kappa"] == float("inf")             # no SI stage yet
    s.step()
    d = s.diagnostics()
    ref = min(O.Oracle(w.n, w.dx, g=w.g, lam=float(w.lam[m]), bc=w.bc).run(w.state(m), cfl=w.cfl, mcfl=w.mcfl,
                                                                            steps=1)[3] for m in range(3))
    # reported to 2^-20 relative, rounded toward zero (its high word)
    assert ref > 0 and -1e-13 * ref <= ref - d["min_kappa"] <= 2.0 ** -19 * ref, (d["min_kappa"], ref)
    s.run_steps(4)
    assert s.diagnostics()["min_kappa"] <= d["min_kappa"]   # running minimum


def test_achieved_cfl_matches_the_dt_rule():
    """after a step, cfl_imex / mcfl are those of the next step: its dt (from
    the current state) times the current maxima over dx"""
    w = W.random_smooth(1024, 4, seed=3, amp=0.1)
    w.cfl, w.mcfl = 2.0, 0.05                          # the material rule binds for some members
    s = gpu_solver(w)
    s.step()
    d = s.diagnostics()
    (h, q, K, Wf), _ = s.get_state(device=False)
    cf, mc = 0.0, 0.0
    for m in range(4):
        dt, nu, um = O.Oracle(w.n, w.dx, lam=float(w.lam[m])).dt([h[m], q[m], K[m], Wf[m]], w.cfl, w.mcfl)
        cf, mc = max(cf, dt * nu / w.dx), max(mc, dt * um / w.dx)
    assert abs(d["cfl_imex"] - cf) <= 1e-13 * cf and abs(d["mcfl"] - mc) <= 1e-13 * mc, (d, cf, mc)
    assert d["cfl_imex"] <= w.cfl * (1 + 1e-14) and d["mcfl"] <= w.mcfl * (1 + 1e-14)
    assert abs(d["mcfl"] - w.mcfl) <= 1e-14 or abs(d["cfl_imex"] - w.cfl) <= 1e-14
