"""Pins of the oracle's Picard re-linearisation of the depth equation (reading
A24).  The paper prints no Picard result, so the fixed
point itself is "parity unpinned"; what is pinned:
  * picard = 0 is the paper's linearised stage (bitwise the default)
  * the passes contract geometrically to a fixed point ("mildly nonlinear")
  * rest state exact, mass conservation, time order 2 preserved
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W

G = 9.81


def test_picard_zero_is_the_linearised_stage():
    w = W.random_smooth(256, 1, seed=7, amp=0.1)
    U = w.state(0)
    a = O.Oracle(w.n, w.dx, lam=1000.0).step(U, 0.01)
    b = O.Oracle(w.n, w.dx, lam=1000.0, picard=0).step(U, 0.01)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_picard_passes_contract_to_a_fixed_point():
    w = W.random_smooth(400, 1, seed=11, amp=0.15)
    U = w.state(0)
    lam = 2000.0
    dt = 2.0 * w.dx / math.sqrt(G * 1.2 + lam / 3)
    S = [O.Oracle(w.n, w.dx, lam=lam, picard=k).stage(U, U, (1 - 1 / math.sqrt(2)) * dt)[0]
         for k in range(6)]
    d = [max(np.max(np.abs(S[k][f] - S[k - 1][f])) for f in range(4)) for k in range(1, 6)]
    scale = max(np.max(np.abs(S[5][f])) for f in range(4))
    assert d[0] > 1e-9                               # the re-linearisation matters
    assert d[1] < 1e-4 * d[0], d                     # contraction (~1e-6 per pass here)
    assert max(d[2:]) < 1e-14 * scale, d             # at the fixed point to round-off


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_picard_rest_state_and_mass(bc):
    n, h0 = 64, 1.1
    h = np.full(n, h0)
    z = np.zeros(n)
    o = O.Oracle(n, 0.1, lam=700.0, bc=(bc, bc), picard=3)
    U = o.step([h, z, h * h, z], 0.01)
    assert np.max(np.abs(U[0] - h)) < 1e-14 and np.max(np.abs(U[1])) < 1e-13   # round-off
    w = W.random_smooth(512, 1, seed=3, amp=0.1, bc=(bc, bc))
    o = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc, picard=2)
    U0 = w.state(0)
    U, *_ = o.run(U0, steps=50)
    assert abs(np.sum(U[0]) - np.sum(U0[0])) <= 1e-13 * np.sum(U0[0])


def test_picard_time_order_two():
    """Halving dt (fixed-dt runs) against a dt/16 reference: order 2 kept."""
    n, lam = 400, 1000.0
    x = W.cell_centres(-50, 50, n)
    U0 = list(W.soliton_state(x, 1.0, 0.2, 0.0, L=100.0))
    o = O.Oracle(n, 100.0 / n, lam=lam, picard=2)
    T = 0.5
    dt0 = 0.02
    ref, *_ = o.run(U0, steps=int(round(T / (dt0 / 16))), dt_fixed=dt0 / 16)
    errs = []
    for k in (1, 2, 4):
        U, *_ = o.run(U0, steps=int(round(T / (dt0 / k))), dt_fixed=dt0 / k)
        errs.append(np.max(np.abs(U[0] - ref[0])))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(orders > 1.8), (errs, orders)
