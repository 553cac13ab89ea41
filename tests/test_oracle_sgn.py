"""Pins of the oracle's classical SGN scheme
against what the paper and the mathematics fix.  CPU only (-m "not gpu").

  * the SGN solitary wave is an EXACT solution of the SGN
    equations: the scheme converges to it at O(dx^2) (a wrong sign, factor or
    the literal g h_{i+1} of P:591 (reading A23) breaks this)
  * one step on a small Fourier mode about rest equals the 2x2 symbol derived
    in tests/linear_theory.py (Rusanov speed, MUSCL, phi system, h*, Heun)
  * rest state exact, mass conservation, the CFL_SGN dt rule
  * hSGN -> SGN as lambda -> infinity: the SI solution approaches
    the SGN solution on the soliton as lambda grows
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests import linear_theory as LT

G = 9.81


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 1)])
def test_sgn_rest_state_is_fixed_point(bc, order, stages):
    n, h0 = 40, 0.8
    h = np.full(n, h0)
    z = np.zeros(n)
    o = O.Oracle(n, 0.05, bc=(bc, bc), order=order)
    U = o.sgn_step([h, z, h * h, z], 0.003, stages=stages)
    assert np.array_equal(U[0], h) and np.array_equal(U[1], z)


def test_sgn_dt_rule():
    n = 8
    h = np.full(n, 2.0)
    q = np.full(n, 2.0 * 0.5)
    o = O.Oracle(n, 0.1)
    assert abs(o.sgn_dt([h, q], 0.9) - 0.9 * 0.1 / (0.5 + math.sqrt(G * 2.0))) < 1e-16


@pytest.mark.parametrize("order,stages", [(2, 2), (1, 2), (2, 1), (1, 1)])
def test_sgn_linearised_step_matches_fourier_symbol(order, stages):
    n, dx, h0 = 64, 0.2, 1.0
    dt = 0.9 * dx / math.sqrt(G * h0)
    o = O.Oracle(n, dx, order=order)
    x = np.arange(n)
    eps = 1e-7
    for k in (2, 8, 16, 24):
        th = 2 * np.pi * k / n
        Gm = LT.sgn_symbol(th, dx, h0, G, dt, order, stages)
        for j in range(2):
            v = np.zeros(2)
            v[j] = 1.0
            pert = eps * np.outer(v, np.cos(th * x))
            U = [h0 + pert[0], pert[1], np.full(n, h0 * h0), np.zeros(n)]
            U2 = o.sgn_step(U, dt, stages=stages)
            resp = np.array([U2[0] - h0, U2[1]])
            pred = eps * np.real(np.outer(Gm[:, j], np.exp(1j * th * x)))
            scale = np.max(np.abs(pred)) + eps * 1e-3
            assert np.max(np.abs(resp - pred)) <= 2e-5 * scale + 1e-15, (k, j)


def _sgn_soliton_err(n, order=2, stages=2, tend=1.0, A=0.2):
    x = W.cell_centres(-50, 50, n)
    U = list(W.soliton_state(x, 1.0, A, 0.0, L=100.0))
    o = O.Oracle(n, 100.0 / n, order=order)
    U, t, s = o.sgn_run(U, cfl=0.9, stages=stages, t_end=tend)
    assert t == tend
    he, _ = W.soliton_exact(x, tend, 1.0, A, 0.0, L=100.0)
    return np.sum(np.abs(U[0] - he)) / np.sum(np.abs(U[0]))


def test_sgn_soliton_second_order_in_dx():
    e = [_sgn_soliton_err(n) for n in (250, 500, 1000, 2000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 1.85), (e, orders)


def test_sgn_soliton_first_order_in_space():
    e = [_sgn_soliton_err(n, order=1) for n in (500, 1000, 2000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 0.8), (e, orders)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_sgn_mass_conservation(bc):
    w = W.random_smooth(512, 1, seed=19, amp=0.1, bc=(bc, bc))
    o = O.Oracle(w.n, w.dx, bc=w.bc)
    U = w.state(0)
    m0 = np.sum(U[0])
    U, t, s = o.sgn_run(U, cfl=0.9, steps=200)
    assert abs(np.sum(U[0]) - m0) <= 1e-13 * m0


def test_hsgn_approaches_sgn_as_lambda_grows():
    """P:113 (lam -> infinity recovers SGN): on the soliton at N = 1000 the SI
    hSGN solution at t = 2 approaches the SGN solution as lam grows from 100
    to 1000 (the O(1/lam) model gap); at this grid larger lam is limited by the
    hSGN discretisation error (1.7e-2 at 5e3, independent of CFL_IMEX)."""
    n = 1000
    x = W.cell_centres(-50, 50, n)
    U0 = list(W.soliton_state(x, 1.0, 0.2, 0.0, L=100.0))
    o = O.Oracle(n, 0.1)
    Us, _, _ = o.sgn_run(U0, cfl=0.9, t_end=2.0)
    d = []
    for lam in (100.0, 300.0, 1000.0):
        oh = O.Oracle(n, 0.1, lam=lam, filter_sigma=0.25)
        Uh, _, _, _ = oh.run(U0, cfl=2.0, mcfl=0.5, t_end=2.0)
        d.append(np.sum(np.abs(Uh[0] - Us[0])) / np.sum(np.abs(Us[0] - 1.0)))
    assert d[0] > d[1] > d[2], d
    assert d[2] < 0.006, d
