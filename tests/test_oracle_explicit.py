"""Pins of the oracle's explicit hSGN scheme
against what the paper and the mathematics fix.  CPU only (-m "not gpu").

  * rest state: every flux constant, every source zero -> exact fixed point
  * SPEC's dt examples for dt = CFL_EX dx / mu_max
  * a spatially uniform state reduces L(U) to the relaxation ODE
    H' = W, W' = -lam (H/h^2 - 1): one step equals the closed-form Euler / Heun
    amplification of that linear ODE (pins the source terms and P:480)
  * one step on a small Fourier mode about rest equals the 4x4 symbol derived
    in tests/linear_theory.py (pins D_x, the pressure coefficients, M, Heun)
  * mass conservation (flux form), the explicit/SI cross-scheme agreement and
    the soliton convergence order
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests import linear_theory as LT

G = 9.81


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 1), (2, 1), (1, 2)])
def test_explicit_rest_state_is_fixed_point(bc, order, stages):
    n, h0 = 40, 1.7
    h = np.full(n, h0)
    z = np.zeros(n)
    o = O.Oracle(n, 0.05, lam=800.0, bc=(bc, bc), order=order)
    U = o.explicit_step([h, z, h * h, z], 0.003, stages=stages)
    for a, b in zip(U, [h, z, h * h, z]):
        assert np.array_equal(a, b)


def test_explicit_dt_spec_examples():
    """u = 0, h = eta = 1, dx = 0.1, CFL = 0.4: dt = 0.4*0.1/3.13209
    at lam = 0 and 0.4*0.1/20.2438 at lam = 1200 (c^2 = g h + lam/3 sigma^2)."""
    n = 16
    h = np.ones(n)
    z = np.zeros(n)
    for lam, dt_ref in ((0.0, 0.012771), (1200.0, 0.0019759)):
        o = O.Oracle(n, 0.1, lam=lam)
        dt, nu, um = o.dt([h, z, h], 0.4, 0.0)
        assert abs(dt - dt_ref) < 1e-6                 # SPEC prints 5 digits
        assert abs(dt - 0.04 / math.sqrt(G + lam / 3.0)) < 1e-15


@pytest.mark.parametrize("stages", [1, 2])
def test_explicit_uniform_state_is_the_relaxation_ode(stages):
    """Uniform h0, q = 0, H = H0, W = W0: all differences vanish, so
    L = (0, 0, W, -lam (H/h0^2 - 1)); with y = (H - h0^2, W), y' = A y,
    A = [[0, 1], [-lam/h0^2, 0]] and one step is (I + dt A [+ (dt A)^2/2]) y."""
    n, h0, lam, dt = 12, 1.3, 900.0, 0.004
    H0, W0 = h0 * h0 * 1.02, 0.07
    o = O.Oracle(n, 0.1, lam=lam)
    h = np.full(n, h0)
    U = o.explicit_step([h, np.zeros(n), np.full(n, H0), np.full(n, W0)], dt, stages=stages)
    A = np.array([[0.0, 1.0], [-lam / h0 ** 2, 0.0]])
    M = np.eye(2) + dt * A + (0.5 * (dt * A) @ (dt * A) if stages == 2 else 0.0)
    y = M @ np.array([H0 - h0 * h0, W0])
    assert np.max(np.abs(U[0] - h0)) == 0 and np.max(np.abs(U[1])) == 0
    assert np.max(np.abs(U[2] - (h0 * h0 + y[0]))) < 1e-14
    assert np.max(np.abs(U[3] - y[1])) < 1e-14


@pytest.mark.parametrize("order,stages", [(2, 2), (1, 2), (2, 1), (1, 1)])
@pytest.mark.parametrize("lam", [0.0, 500.0, 2e4])
def test_explicit_linearised_step_matches_fourier_symbol(order, stages, lam):
    n, dx, h0 = 64, 0.2, 1.0
    dt = 0.4 * dx / math.sqrt(G * h0 + lam / 3)
    o = O.Oracle(n, dx, lam=lam, order=order)
    x = np.arange(n)
    eps = 1e-7
    for k in (2, 8, 16, 24):
        th = 2 * np.pi * k / n
        Gm = LT.explicit_symbol(th, dx, h0, lam, G, dt, order, stages)
        for j in range(4):
            v = np.zeros(4)
            v[j] = 1.0
            pert = eps * np.outer(v, np.cos(th * x))
            U = [h0 + pert[0], pert[1], h0 * h0 + pert[2], pert[3]]
            U2 = o.explicit_step(U, dt, stages=stages)
            resp = np.array([U2[0] - h0, U2[1], U2[2] - h0 * h0, U2[3]])
            pred = eps * np.real(np.outer(Gm[:, j], np.exp(1j * th * x)))
            scale = np.max(np.abs(pred)) + eps * 1e-3
            assert np.max(np.abs(resp - pred)) <= 2e-5 * scale + 1e-15, (k, j)


def test_explicit_symbol_stability_envelope():
    """S:738 / P:631: Heun at CFL_EX = 1.2 grows strongly at grid scale
    (rho ~ 1.1 per step), at the paper's 0.4 only ~1.001 (<= 1 + 1e-5 with the
    A19 filter).  Reading A22: forward Euler (the literal first-order scheme of
    P:444) is unstable at every CFL (rho = |1 + i dt omega| > 1; 1.08 at 0.4)."""
    dx, h0, lam = 0.1, 1.0, 1000.0
    c = math.sqrt(G * h0 + lam / 3)
    assert LT.explicit_max_growth(dx, h0, lam, G, 1.2 * dx / c) > 1.05
    assert LT.explicit_max_growth(dx, h0, lam, G, 0.4 * dx / c) < 1.002
    assert LT.explicit_max_growth(dx, h0, lam, G, 0.4 * dx / c, filter_sigma=0.25) < 1.00001
    assert LT.explicit_max_growth(dx, h0, lam, G, 0.4 * dx / c, order=1, stages=1) > 1.07
    assert LT.explicit_max_growth(dx, h0, lam, G, 0.1 * dx / c, order=1, stages=1) > 1.004


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_explicit_mass_conservation(bc):
    w = W.random_smooth(512, 1, seed=9, amp=0.1, bc=(bc, bc))
    o = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc)
    U = w.state(0)
    m0 = np.sum(U[0])
    U, t, s = o.explicit_run(U, cfl=0.4, steps=200)
    assert abs(np.sum(U[0]) - m0) <= 1e-13 * m0


def test_explicit_and_si_agree_on_the_soliton():
    """Both schemes discretise the same hSGN system: on the cfg1
    soliton at N = 1000 the second-order solutions at t = 2 differ by far less
    than either differs from the initial data."""
    w = W.cfg1()
    lam = float(w.lam[0])
    o = O.Oracle(w.n, w.dx, lam=lam)
    U0 = w.state(0)
    Ue, te, _ = o.explicit_run(U0, cfl=0.4, t_end=2.0)
    Us, ts, _, _ = o.run(U0, cfl=2.0, mcfl=0.5, t_end=2.0)
    assert te == 2.0 and ts == 2.0
    d = np.sum(np.abs(Ue[0] - Us[0])) / np.sum(np.abs(Us[0] - 1.0))
    moved = np.sum(np.abs(U0[0] - Us[0])) / np.sum(np.abs(Us[0] - 1.0))
    assert d < 0.02 and moved > 1.0, (d, moved)


def _explicit_soliton_err(n, lam, order=2, stages=2, tend=1.0, sigma=0.0):
    x = W.cell_centres(-50, 50, n)
    U = list(W.soliton_state(x, 1.0, 0.2, 0.0, L=100.0))
    o = O.Oracle(n, 100.0 / n, lam=lam, order=order, filter_sigma=sigma)
    U, t, s = o.explicit_run(U, cfl=0.4, stages=stages, t_end=tend)
    he, _ = W.soliton_exact(x, tend, 1.0, 0.2, 0.0, L=100.0)
    return np.sum(np.abs(U[0] - he)) / np.sum(np.abs(U[0]))


@pytest.mark.slow
def test_explicit_soliton_second_order_in_dx():
    """Heun + MUSCL with the A19 filter (the literal scheme blows up under flow,
    reading A22) converges at second order on the soliton."""
    e = [_explicit_soliton_err(n, 5000.0, sigma=0.25) for n in (1000, 2000, 4000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 1.7), (e, orders)


def test_explicit_soliton_first_order_in_space():
    """Order-1 faces (Heun in time; forward Euler is unstable, A22): O(dx)."""
    e = [_explicit_soliton_err(n, 5000.0, order=1, stages=2) for n in (500, 1000, 2000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 0.8), (e, orders)


def test_literal_explicit_scheme_grows_under_flow_and_the_filter_tames_it():
    """Reading A22: about a uniform flow u0 = 0.3 the literal scheme (Heun,
    unlimited MUSCL, alpha = |u|) amplifies seeded noise by ~1.04 per step at
    CFL_EX = 0.4; with the A19 filter the growth is below 1.003 per step."""
    n, dx, h0, lam, u0 = 256, 0.05, 1.0, 1000.0, 0.3
    dt = 0.4 * dx / (u0 + math.sqrt(G * h0 + lam / 3))
    rng = np.random.default_rng(1)
    rates = []
    for sigma in (0.0, 0.25):
        h = h0 + 1e-12 * rng.standard_normal(n)
        U = [h, h * u0, h * h, np.zeros(n)]
        o = O.Oracle(n, dx, lam=lam, filter_sigma=sigma)
        U, _, _ = o.explicit_run(U, steps=300, dt_fixed=dt)
        a1 = np.max(np.abs(U[0] - np.mean(U[0])))
        U, _, _ = o.explicit_run(U, steps=200, dt_fixed=dt)
        a2 = np.max(np.abs(U[0] - np.mean(U[0])))
        rates.append((a2 / a1) ** (1 / 200))
    assert rates[0] > 1.03 and rates[1] < 1.003, rates
