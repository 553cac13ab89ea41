"""Pins of the CPU oracle (oracle/hsgn_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself.  CPU only (-m "not gpu").

Each test names the passage / closed form it pins; DESIGN.md section 4 maps
oracle functions to the pins that cover them."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests import linear_theory as LT

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G = 9.81


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                yield line.split()


# --------------------------------------------------------------------------
# Tableau
# --------------------------------------------------------------------------
def test_tableau_order_conditions_and_weights():
    T = O.paper_tableau()
    gold = {k: float(v) for k, v in _rows("tableau.txt")}
    g = T.aI[0][0]
    assert abs(g - gold["gamma"]) < 1e-16
    assert abs(T.aE[1][0] - gold["c"]) < 4e-16
    b = np.array([T.b[0], T.b[1]])
    cE = np.array([0.0, T.aE[1][0]])
    cI = np.array([T.aI[0][0], T.aI[1][0] + T.aI[1][1]])
    assert abs(b.sum() - 1) < 1e-15                 # sum b = 1
    assert abs(b @ cE - 0.5) < 1e-15                # second order, explicit
    assert abs(b @ cI - 0.5) < 1e-15                # second order, implicit
    assert T.aI[1][0] == T.b[0] and T.aI[1][1] == T.b[1]   # stiffly accurate
    wE, wR = O.tableau_weights(T)
    assert abs(wE - gold["wE"]) < 4e-15 and abs(wE - (3 + 2 * math.sqrt(2))) < 4e-15
    assert abs(wR - gold["wR"]) < 4e-15 and abs(wR - (1 + math.sqrt(2))) < 4e-15


def test_tableau_validation_rejects_non_stiffly_accurate():
    T = O.make_tableau(2, [[0, 0], [1.0, 0]], [[0.5, 0], [0.25, 0.5]], [0.5, 0.5])
    with pytest.raises(O.OracleError):
        O.tableau_weights(T)


# --------------------------------------------------------------------------
# Pointwise algebra and the dt rule
# --------------------------------------------------------------------------
def test_pointwise_spec_examples():
    for kind, g, lam, h, eta, e1, e2, exp, dig, cite in _rows("spec_pointwise.txt"):
        g, lam, h, eta, e1, e2, exp = map(float, (g, lam, h, eta, e1, e2, exp))
        tol = 0.5 * 10.0 ** (-int(dig)) + 1e-13
        H = h * eta
        if kind == "celerity":
            got = O.celerity(g, lam, h, H)
        elif kind == "alpha":
            got = O.coeffs(g, lam, 0.0, h, H, H)["alpha"]
        elif kind == "a2":
            got = O.coeffs(g, lam, 0.0, h, H, H)["a2"]
        elif kind == "dt_cfl":
            o = O.Oracle(8, e1, g=g, lam=lam)
            U = [np.full(8, h), np.zeros(8), np.full(8, H), np.zeros(8)]
            got = o.dt(U, e2, 0.5)[0]
        else:
            raise AssertionError(kind)
        assert abs(got - exp) <= tol, (kind, cite, got, exp)


def test_dt_rule_material_branch():
    # dx = 0.1, u_max = 2, MCFL = 0.75, eigenvalue constraint slack -> 0.0375
    o = O.Oracle(8, 0.1, lam=1.0)
    U = [np.ones(8), np.full(8, 2.0), np.ones(8), np.zeros(8)]
    dt, nu, um = o.dt(U, 50.0, 0.75)
    assert um == 2.0 and abs(dt - 0.0375) < 1e-15
    # u_max = 0 -> material rule inactive
    U0 = [np.ones(8), np.zeros(8), np.ones(8), np.zeros(8)]
    dt0, nu0, _ = o.dt(U0, 2.0, 0.5)
    assert abs(dt0 - 2.0 * 0.1 / math.sqrt(9.81 + 1 / 3)) < 1e-15


def test_nu_max_reading_against_paper_cfl_sw():
    """P:703 prints CFL_SW implied by CFL_IMEX = 2 on the Gaussian bell.  The
    c^2 = gh + (lam/3)(eta/h)^2 reading (A7) reproduces 0.66/0.48/0.22 (and 1.22
    vs the printed 1.34 at lam = 100); P:628's literal form would give 2.0."""
    w = W.gaussian_bell()
    x = w.x()
    for lam, paper, cite in _rows("paper_p703_cfl_sw.txt"):
        lam, paper = float(lam), float(paper)
        o = O.Oracle(w.n, w.dx, lam=lam, bc=w.bc)
        dt, nu, um = o.dt(w.state(0), 2.0, 0.5)
        cfl_sw = dt * np.max(np.abs(w.q[0] / w.h[0]) + np.sqrt(G * w.h[0])) / w.dx
        assert abs(cfl_sw - paper) / paper < 0.10, (lam, cfl_sw, paper)
        assert abs(cfl_sw - 2.0) > 0.5
    del x


def test_kappa_equilibrium_closed_form():
    """At eta = h, W = 0 (so H^dagger = h^2 + lam tau^2 by P:502-503):
    beta = g h + (2 lam / 3) h^2 / (h^2 + lam tau^2)  (A16 / SURVEY A.3),
    and beta > 0."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        h = rng.uniform(0.05, 3.0)
        lam = 10 ** rng.uniform(0, 5)
        tau = 10 ** rng.uniform(-4, -1)
        c = O.coeffs(G, lam, tau, h, h * h, h * h + lam * tau * tau)
        ref = G * h + (2 * lam / 3) * h * h / (h * h + lam * tau * tau)
        scale = abs(c["a2"]) + abs(c["beta"] - c["a2"])   # cancellation in P:507
        assert abs(c["beta"] - ref) <= 2e-15 * scale
        assert c["beta"] > 0
        # b1 identity: 1/beta1 = h^2/(h^2 + lam tau^2); dh b1
        assert abs(1 / c["beta1"] - h * h / (h * h + lam * tau * tau)) < 1e-14
        b1 = 1 / c["beta1"]
        assert abs(c["beta2"] - 2 * lam * tau * tau / h ** 3 * b1 * b1) <= 1e-13 * abs(c["beta2"]) + 1e-300


def test_pressure_gradient_split_identity():
    """p_x = a^2 h_x + lam alpha (h eta)_x for smooth fields, with
    p = g h^2/2 + (lam/3) eta (1 - eta/h).  Checked by centred
    differences of p (independent of the oracle's coefficient formulas): O(dx^2)."""
    errs = []
    for n in (200, 400, 800):
        x = np.linspace(0, 1, n + 1)
        h = 1 + 0.3 * np.sin(2 * np.pi * x)
        eta = h * (1 + 0.05 * np.cos(2 * np.pi * x))
        lam = 300.0
        p = G * h * h / 2 + lam / 3 * eta * (1 - eta / h)
        dx = x[1] - x[0]
        px = (p[2:] - p[:-2]) / (2 * dx)
        hx = (h[2:] - h[:-2]) / (2 * dx)
        Hx = ((h * eta)[2:] - (h * eta)[:-2]) / (2 * dx)
        rhs = []
        for i in range(1, n):
            c = O.coeffs(G, lam, 0.0, h[i], h[i] * eta[i], h[i] * eta[i])
            rhs.append(c["a2"] * hx[i - 1] + lam * c["alpha"] * Hx[i - 1])
        errs.append(np.max(np.abs(px - np.array(rhs))))
    assert errs[1] < errs[0] / 3.5 and errs[2] < errs[1] / 3.5


# --------------------------------------------------------------------------
# Tridiagonal solve (A3): dense LU as the pin
# --------------------------------------------------------------------------
@pytest.mark.parametrize("cyclic", [False, True])
def test_thomas_matches_dense_lu(cyclic):
    rng = np.random.default_rng(11)
    for n in list(range(3, 9)) + [17, 64]:
        for _ in range(20):
            lo = -rng.uniform(0, 1, n)
            up = -rng.uniform(0, 1, n)
            di = 1 + np.abs(lo) + np.abs(up) + rng.uniform(0, 1, n)
            rhs = rng.standard_normal(n)
            A = np.diag(di)
            for i in range(n):
                if i > 0:
                    A[i, i - 1] = lo[i]
                if i < n - 1:
                    A[i, i + 1] = up[i]
            if cyclic:
                A[0, n - 1] += lo[0]
                A[n - 1, 0] += up[n - 1]
            ref = np.linalg.solve(A, rhs)
            got = O.thomas(lo, di, up, rhs, cyclic=cyclic)
            assert np.max(np.abs(got - ref)) <= 1e-12 * (1 + np.max(np.abs(ref)))


def test_thomas_spec_examples():
    # S:173-175
    x = O.thomas([0, -1, -1], [2, 2, 2], [-1, -1, 0], [1, 0, 1])
    assert np.max(np.abs(x - 1.0)) < 1e-15
    with pytest.raises(O.OracleError) as e:
        O.thomas([-1, -1, -1], [2, 2, 2], [-1, -1, -1], [0, 0, 0], cyclic=True)
    assert e.value.status in (O.E_SINGULAR,)


# --------------------------------------------------------------------------
# Fixed points and worked stage examples
# --------------------------------------------------------------------------
@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order", [1, 2])
def test_rest_state_is_fixed_point(bc, order):
    """(h0, 0, h0^2, 0) is an exact fixed point of both stages (P:502-515:
    W^dagger = lam tau, H^dagger = h0^2 + lam tau^2, hbar = h0, Hbar = h0^2, Wbar = 0)."""
    for h0, lam, dt in [(1.0, 500.0, 0.05), (0.4, 1e5, 1e-3), (2.0, 0.0, 0.1), (1.3, 1e4, 0.02)]:
        n = 32
        o = O.Oracle(n, 0.2, lam=lam, bc=(bc, bc), order=order)
        U = [np.full(n, h0), np.zeros(n), np.full(n, h0 * h0), np.zeros(n)]
        U2 = o.step(U, dt)
        assert np.max(np.abs(U2[0] - h0)) <= 4e-15 * h0
        assert np.max(np.abs(U2[2] - h0 * h0)) <= 8e-15 * h0 * h0
        scale = max(1.0, lam * dt)           # round-off of W^dagger = lam tau + ...
        assert np.max(np.abs(U2[1])) <= 1e-14 * scale * 20 and np.max(np.abs(U2[3])) <= 1e-14 * scale * 20


def test_stage_worked_examples_uniform_state():
    """S:406 (H~ = (h eta)* + tau (hw)* + lam tau^2 = 2 for 1, 0, 1) and S:428
    (hbar = 1, (h eta)^dagger = 1.5, lam tau^2 = 0.5 -> hbar eta = 1.0) through
    a uniform u = 0 state (predictor = identity)."""
    n = 16
    tau = 0.5
    lam = 0.5 / tau ** 2                 # lam tau^2 = 0.5
    o = O.Oracle(n, 0.1, lam=lam)
    U = [np.ones(n), np.zeros(n), np.ones(n), np.zeros(n)]   # H^dagger = 1 + 0 + 0.5
    out, _ = o.stage(U, U, tau)
    assert np.max(np.abs(out[0] - 1.0)) < 2e-14
    assert np.max(np.abs(out[2] - 1.0)) < 2e-14              # 1.5 / (1 + 0.5)
    assert np.max(np.abs(out[3])) < 5e-14                    # lam tau - lam tau * 1
    lam = 1.0 / tau ** 2                 # lam tau^2 = 1, (h eta)* = 1 -> H~ = 2
    o = O.Oracle(n, 0.1, lam=lam)
    out, _ = o.stage(U, U, tau)
    assert np.max(np.abs(out[2] - 2.0 / (1.0 + 1.0))) < 2e-14


# --------------------------------------------------------------------------
# Conservation
# --------------------------------------------------------------------------
@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_mass_conservation(bc):
    w = W.random_smooth(256, 1, seed=5, amp=0.1)
    o = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=(bc, bc))
    U0 = w.state(0)
    m0 = O.mass(U0[0], w.dx)
    U, t, s, mb = o.run(U0, cfl=2.0, mcfl=0.5, steps=40)
    assert mb > 0
    assert abs(O.mass(U[0], w.dx) - m0) <= 2e-14 * m0


def test_wall_equals_mirrored_periodic():
    """A wall (A10: h, K, W even, q odd, Neumann depth rows) on [0, L] must equal
    the periodic solution on the mirror-doubled domain [-L, L]."""
    w = W.random_smooth(64, 1, seed=9, amp=0.1)
    h, q, K, Wf = w.state(0)
    n = w.n
    o_wall = O.Oracle(n, w.dx, lam=700.0, bc=("wall", "wall"))
    dbl = [np.concatenate([f[::-1] * s, f]) for f, s in zip((h, q, K, Wf), (1, -1, 1, 1))]
    o_per = O.Oracle(2 * n, w.dx, lam=700.0, bc=("periodic", "periodic"))
    Uw = [h, q, K, Wf]
    Up = dbl
    for _ in range(10):
        Uw = o_wall.step(Uw, 0.02)
        Up = o_per.step(Up, 0.02)
    for a, b in zip(Uw, Up):
        assert np.max(np.abs(a - b[n:])) <= 1e-12 * (1 + np.max(np.abs(b)))


def test_flat_bathymetry_is_bitwise_flat():
    w = W.random_smooth(64, 1, seed=2)
    o0 = O.Oracle(w.n, w.dx, lam=900.0)
    o1 = O.Oracle(w.n, w.dx, lam=900.0, b=np.zeros(w.n))
    a = o0.step(w.state(0), 0.01)
    b = o1.step(w.state(0), 0.01)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


# --------------------------------------------------------------------------
# Linearised step symbol (whole linear stage, derived in
# tests/linear_theory.py from P:500-517 and P:397-403)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 2), (2, 1), (1, 1)])
@pytest.mark.parametrize("lam", [0.0, 500.0, 2e4])
def test_linearised_step_matches_fourier_symbol(order, stages, lam):
    n, dx, h0 = 64, 0.2, 1.0
    dt = 2.5 * dx / math.sqrt(G * h0 + lam / 3)
    T = O.paper_tableau() if stages == 2 else O.euler_tableau()
    o = O.Oracle(n, dx, lam=lam, order=order, tableau=T)
    x = np.arange(n)
    eps = 1e-7
    for k in (2, 8, 16, 24):
        th = 2 * np.pi * k / n
        Gm = LT.step_symbol(th, dx, h0, lam, G, dt, order, stages)
        for j in range(4):
            v = np.zeros(4)
            v[j] = 1.0
            pert = eps * np.outer(v, np.cos(th * x))
            U = [h0 + pert[0], pert[1], h0 * h0 + pert[2], pert[3]]
            U2 = o.step(U, dt)
            resp = np.array([U2[0] - h0, U2[1], U2[2] - h0 * h0, U2[3]])
            pred = eps * np.real(np.outer(Gm[:, j], np.exp(1j * th * x)))
            scale = np.max(np.abs(pred)) + eps * 1e-3
            assert np.max(np.abs(resp - pred)) <= 2e-5 * scale + 1e-15, (k, j)


def test_seeded_rest_growth_matches_symbol_and_filter_removes_it():
    """Reading A19: about flat rest the literal scheme amplifies grid-scale noise
    by max_theta rho(G) per step (1.07 at lam = 500, dx = 0.2, CFL_IMEX = 2.7);
    the A19 filter (sigma = 0.25 on q and W) makes every mode non-growing."""
    n, dx, h0, lam = 256, 0.2, 1.0, 500.0
    dt = 2.7 * dx / math.sqrt(G * h0 + lam / 3)
    rho = LT.max_growth(dx, h0, lam, G, dt)
    assert 1.05 < rho < 1.09
    assert LT.max_growth(dx, h0, lam, G, dt, filter_sigma=0.25) <= 1.0 + 1e-12
    w = W.flat_rest(n, dx, h0, lam, noise=1e-13, seed=1)
    o = O.Oracle(n, dx, lam=lam)
    U = w.state(0)
    U, *_ = o.run(U, steps=150, dt_fixed=dt)
    a1 = np.max(np.abs(U[1]))
    U, *_ = o.run(U, steps=100, dt_fixed=dt)
    a2 = np.max(np.abs(U[1]))
    growth = (a2 / a1) ** (1 / 100)
    assert abs(growth - rho) / rho < 0.01
    of = O.Oracle(n, dx, lam=lam, filter_sigma=0.25)
    U = w.state(0)
    U, *_ = of.run(U, steps=250, dt_fixed=dt)
    assert np.max(np.abs(U[1])) < 1e-11


# --------------------------------------------------------------------------
# Dispersion: the scheme's phase speed converges to the hSGN slow branch
# (derived from P:101-111) at second order; the branch itself is O(1/lam)
# from SGN's.
# --------------------------------------------------------------------------
def test_dispersion_converges_to_hsgn_branch():
    h0, lam, L = 1.0, 1000.0, 20.0
    k = 2 * np.pi / L * 1      # k h0 = 0.314
    om = LT.hsgn_slow_omega(k, h0, lam, G)
    assert abs(om / LT.sgn_omega(k, h0, G) - 1) < 1e-3   # O(1/lam) model gap
    Tend = 0.5 * L / (om / k)
    errs = []
    for n in (50, 100, 200):
        dx = L / n
        x = W.cell_centres(0, L, n)
        U = list(LT.slow_mode_state(x, k, 1e-6, h0, lam, G))
        o = O.Oracle(n, dx, lam=lam, filter_sigma=0.0)
        nsteps = 8 * n // 50 * 5
        U, t, s, _ = o.run(U, steps=nsteps, dt_fixed=Tend / nsteps)
        hp = U[0] - h0
        c = np.sum(hp * np.exp(-1j * k * x))
        phase = -np.angle(c)          # = omega_num * T (mod 2pi)
        om_num = phase / Tend
        errs.append(abs(om_num - om) / om)
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(orders > 1.8), (errs, orders)


# --------------------------------------------------------------------------
# SGN solitary wave: second order in dx (order 2), first order
# (SI Euler + order 1), error decreasing with lambda.
# --------------------------------------------------------------------------
def _soliton_err(n, lam, A=0.2, order=2, tableau=None, cfl=2.0, tend=1.0):
    x = W.cell_centres(-50, 50, n)
    U = list(W.soliton_state(x, 1.0, A, 0.0, L=100.0))
    o = O.Oracle(n, 100.0 / n, lam=lam, order=order, tableau=tableau)
    U, t, s, mb = o.run(U, cfl=cfl, mcfl=0.5, t_end=tend)
    assert abs(t - tend) < 1e-12 and mb > 0
    he, _ = W.soliton_exact(x, tend, 1.0, A, 0.0, L=100.0)
    return np.sum(np.abs(U[0] - he)) / np.sum(np.abs(U[0]))


@pytest.mark.slow
def test_soliton_second_order_in_dx():
    e = [_soliton_err(n, 5000.0) for n in (1000, 2000, 4000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 1.7), (e, orders)


def test_soliton_first_order_scheme():
    e = [_soliton_err(n, 5000.0, order=1, tableau=O.euler_tableau()) for n in (500, 1000, 2000)]
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 0.8), (e, orders)


@pytest.mark.slow
def test_soliton_error_decreases_with_lambda():
    e = [_soliton_err(4000, lam) for lam in (100.0, 500.0, 1000.0, 5000.0)]
    assert all(a > b for a, b in zip(e[:-1], e[1:])), e


def test_time_order_two():
    """Halving dt at fixed grid (fixed dt runs) -> order 2 against a dt/16 run."""
    n, lam = 400, 1000.0
    x = W.cell_centres(-50, 50, n)
    U0 = list(W.soliton_state(x, 1.0, 0.2, 0.0, L=100.0))
    o = O.Oracle(n, 100.0 / n, lam=lam)
    T = 0.5
    ref, *_ = o.run(U0, steps=320, dt_fixed=T / 320)
    e = []
    for s in (10, 20, 40):
        U, *_ = o.run(U0, steps=s, dt_fixed=T / s)
        e.append(np.max(np.abs(U[0] - ref[0])))
    orders = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(orders > 1.8), (e, orders)


# --------------------------------------------------------------------------
# Bathymetry (A9): lake at rest exact at lam = 0, O(dx^2) at lam > 0
# --------------------------------------------------------------------------
def test_lake_at_rest_exact_lambda0():
    w = W.lake_at_rest(128, 0.0)
    o = O.Oracle(w.n, w.dx, lam=0.0, b=w.b)
    U, *_ = o.run(w.state(0), steps=20, dt_fixed=0.02)
    assert np.max(np.abs(U[1])) < 1e-13
    assert np.max(np.abs(U[0] - w.h[0])) < 1e-13


def test_lake_at_rest_second_order_lambda_positive():
    errs = []
    for n in (256, 512, 1024):
        w = W.lake_at_rest(n, 1e4)
        o = O.Oracle(w.n, w.dx, lam=1e4, b=w.b)
        U, t, s, _ = o.run(w.state(0), cfl=2.0, mcfl=0.5, t_end=0.05)
        errs.append(np.max(np.abs(U[1] / U[0])))
    orders = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(orders > 1.8), (errs, orders)


def test_soliton_mass_closed_form():
    (n, m, tol, cite), = list(_rows("soliton_mass.txt"))
    n = int(n)
    x = W.cell_centres(-50, 50, n)
    h, *_ = W.soliton_state(x, 1.0, 1.0, 0.0)
    kappa = math.sqrt(3 / 8)
    exact = 100 + 2 / kappa * math.tanh(50 * kappa)
    assert abs(exact - float(m)) < 1e-8
    assert abs(O.mass(h, 100.0 / n) - exact) < float(tol)


# --------------------------------------------------------------------------
# Rusanov face flux (P:466 with alpha = max(|u-|, |u+|), A4): hand arithmetic
# --------------------------------------------------------------------------
def test_rusanov_face_hand_example():
    # h- = h+ = 1, q- = 1, q+ = 3 (u- = 1, u+ = 3, alpha = 3),
    # H- = H+ = 2, W- = 0, W+ = 1:
    #   F^q = 1/2 (1*1 + 3*3) - 1/2*3*(3-1) = 2
    #   F^H = 1/2 (2*1 + 2*3) - 0           = 4
    #   F^W = 1/2 (0*1 + 1*3) - 1/2*3*(1-0) = 0
    F = O.rusanov_face([1.0, 1.0, 2.0, 0.0], [1.0, 3.0, 2.0, 1.0])
    assert F[0] == 2.0 and F[1] == 4.0 and F[2] == 0.0
    # consistency: equal states -> physical flux
    F = O.rusanov_face([2.0, -1.0, 5.0, 3.0], [2.0, -1.0, 5.0, 3.0])
    assert np.allclose(F, [0.5, -2.5, -1.5], rtol=0, atol=1e-15)


# --------------------------------------------------------------------------
# Consistency of one stage with the PDE: as tau -> 0 the
# stage tendency (U_new - U)/tau is the semi-discrete right-hand side, which
# must converge at O(dx^2) to the hSGNb equations evaluated analytically
# (spectral derivatives of smooth periodic fields; independent of the oracle).
# --------------------------------------------------------------------------
def _spectral_dx(f, L):
    n = len(f)
    k = 2 * np.pi * np.fft.fftfreq(n, d=L / n)
    return np.real(np.fft.ifft(1j * k * np.fft.fft(f)))


@pytest.mark.parametrize("lam,with_b", [(0.0, True), (300.0, False), (300.0, True)])
def test_stage_tendency_converges_to_hsgnb_pde(lam, with_b):
    L = 10.0
    kx = 2 * np.pi / L
    errs = []
    for n in (64, 128, 256):
        x = W.cell_centres(0, L, n)
        h = 1 + 0.2 * np.sin(kx * x)
        u = 0.1 + 0.3 * np.cos(kx * x)
        eta = h * (1 + 0.01 * np.sin(2 * kx * x))
        w = 0.05 * np.cos(kx * x)
        b = 0.1 * np.sin(kx * x + 0.3) if with_b else np.zeros(n)
        etat = eta + 1.5 * b
        U = [h, h * u, h * etat, h * w]
        pt = lam / 3 * (1 - eta / h)                          # p~
        rhs = [-_spectral_dx(h * u, L),
               -_spectral_dx(h * u * u + 0.5 * G * h * h + eta * pt, L)
               - (G * h + 1.5 * pt) * _spectral_dx(b, L),
               -_spectral_dx(h * u * etat, L) + h * w,
               -_spectral_dx(h * u * w, L) + 3 * pt]
        o = O.Oracle(n, L / n, lam=lam, b=b if with_b else None)
        tau = 1e-9         # O(tau lam) stiff terms below the O(dx^2) error
        out, _ = o.stage(U, U, tau)
        e = [np.max(np.abs((out[k] - U[k]) / tau - rhs[k])) / (np.max(np.abs(rhs[k])) + 1e-3)
             for k in range(4)]
        errs.append(e)
    errs = np.array(errs)
    orders = np.log2(errs[:-1] / errs[1:])
    assert np.all(errs[-1] < 5e-3), errs
    assert np.all(orders > 1.7), (errs, orders)


# --------------------------------------------------------------------------
# Wavemaker and sponge relaxation zones (A10; cfg4)
# --------------------------------------------------------------------------
def _airy(omega, h0):
    k = 1.0
    for _ in range(200):
        k = omega ** 2 / (G * np.tanh(k * h0))
    return k, omega / k


def _channel(n=2000, L=40.0, h0=0.4, lam=1000.0, amp=0.001, period=2.02, sponge=True, b=None):
    omega = 2 * np.pi / period
    k, cp = _airy(omega, h0)
    relax = dict(x_min=0.0, level=h0, gen_x1=4.0, gen_rate=0.1, amp=amp, omega=omega, k=k, cp=cp,
                 sp_x0=30.0, sp_rate=0.1 if sponge else 0.0)
    o = O.Oracle(n, L / n, lam=lam, bc=("transmissive", "transmissive"), b=b, relax=relax,
                 filter_sigma=0.25)
    bb = np.zeros(n) if b is None else b
    h = h0 - bb
    U = [h, np.zeros(n), h * (h + 1.5 * bb), np.zeros(n)]
    return o, U, omega


def test_wavemaker_zero_amplitude_keeps_rest():
    o, U, _ = _channel(n=400, amp=0.0)
    U2, t, s, _ = o.run(U, cfl=2.0, mcfl=0.5, t_end=4.0)
    assert np.max(np.abs(U2[0] - U[0])) < 1e-12 and np.max(np.abs(U2[1])) < 1e-12   # round-off only


def test_sponge_keeps_lake_at_rest_over_bathymetry():
    n, L = 400, 40.0
    x = W.cell_centres(0, L, n)
    b = 0.1 * np.exp(-((x - 35.0) / 2.0) ** 2)
    relax = dict(x_min=0.0, level=0.4, sp_x0=30.0, sp_rate=0.1)
    o = O.Oracle(n, L / n, lam=0.0, bc=("wall", "wall"), b=b, relax=relax)
    h = 0.4 - b
    U = [h, np.zeros(n), h * (h + 1.5 * b), np.zeros(n)]
    U2, *_ = o.run(U, steps=20, dt_fixed=0.01)
    assert np.max(np.abs(U2[0] - h)) < 1e-13 and np.max(np.abs(U2[1])) < 1e-13


def _solve_k(omega, h0, lam):
    lo, hi = 1e-4, 50.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if LT.hsgn_slow_omega(mid, h0, lam, G) < omega:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_wavemaker_generates_the_hsgn_wavelength():
    """The wavemaker zone (A10) radiates waves whose wavelength beyond the zone is
    the hSGN one at the forcing frequency (slow branch, derived from P:101-111),
    within 3 %; the sponge removes most of the wave before x = 40."""
    h0, lam = 0.4, 1000.0
    o, U, omega = _channel(h0=h0, lam=lam)
    U2, t, s, _ = o.run(U, cfl=2.0, mcfl=0.5, t_end=10.0)
    x = W.cell_centres(0, 40.0, 2000)
    eta = U2[0] - h0
    sel = (x > 5.0) & (x < 15.0)
    xs, es = x[sel], eta[sel]
    zc = xs[1:][np.sign(es[1:]) != np.sign(es[:-1])]
    lam_num = 2.0 * np.mean(np.diff(zc))
    lam_th = 2 * np.pi / _solve_k(omega, h0, lam)
    assert abs(lam_num - lam_th) / lam_th < 0.03, (lam_num, lam_th)
    inner = np.max(np.abs(eta[(x > 6) & (x < 14)]))
    assert inner > 0.5 * 0.001                     # a wave of the forced amplitude
    tail = np.max(np.abs(eta[x > 38]))
    assert tail < 0.2 * inner, (tail, inner)
