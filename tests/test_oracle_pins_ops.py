"""Pins of the oracle's operator-split extras and of the Picard pass, against
closed forms and independent solves -- never against the oracle itself.
CPU only (-m "not gpu").

The A19 filter and the A10 relaxation zones run after the step
(hsgn_oracle.c orc_step_t).  With the one-stage tableau and dt = 0 the SI stage
is the identity bit for bit (tau = 0: no fluxes, rho = mu = 0, Hbar = H^dag,
Wbar = W^dag), so orc_step_t(t, dt = 0) = relax(filter(U), t) exactly: the two
operators are observable on their own.

* A19 filter (A19): on a single Fourier mode
  e^{i j theta} the stencil f - (sigma/16)(f_{-2} - 4 f_{-1} + 6 f - 4 f_{+1} + f_{+2})
  multiplies the mode by 1 - sigma sin^4(theta/2) (the fourth difference has the
  symbol (2 - 2 cos theta)^2 = 16 sin^4(theta/2)); only q and W (mask) change;
  a wall equals the mirror-doubled periodic domain with q odd.  The filtered
  one-step response equals LT.step_symbol(..., filter_sigma).
* A10 relaxation zones: U <- U - s(x)(U - U_target(x, t)) with the ramps and
  targets as written in DESIGN.md A10 (the reading itself); the wavemaker
  target is a right-going linear wave, u = c_p eta / h0.
* A24 Picard pass: its fixed point is the solution of the UN-frozen
  eliminated depth equation (P:268-285 with b1 = h^2/(h^2 + lam tau^2) and
  d b1/dh evaluated at h^{n+1} instead of h^n), discretised as P:500-512
  (reading A1); on a state at rest in u, eta = h, w = 0 the predictor is
  closed-form (q^dag = 0, H^dag = h^2 + lam tau^2), so the equation is solved
  here by dense Newton in numpy with no oracle code.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests import linear_theory as LT

G = 9.81


def _split_ops(o, U, t=0.0):
    """relax(filter(U), t) of the oracle: orc_step_t with the 1-stage tableau, dt = 0."""
    o.T = O.euler_tableau()
    return o.step(U, 0.0, t=t)


def _smooth_state(n, seed, amp=0.05):
    rng = np.random.default_rng(seed)
    x = np.arange(n) / n
    h = 1.0 + amp * np.cos(2 * np.pi * x + rng.uniform(0, 6))
    q = 0.1 * np.sin(2 * np.pi * 2 * x + rng.uniform(0, 6))
    K = h * h * (1.0 + 0.01 * np.cos(2 * np.pi * 3 * x))
    Wf = 0.02 * np.cos(2 * np.pi * x + rng.uniform(0, 6))
    return [h, q, K, Wf]


# --------------------------------------------------------------------------
# A19 filter
# --------------------------------------------------------------------------
def test_split_ops_identity_without_filter_or_relaxation():
    n = 48
    U = _smooth_state(n, 1)
    out = _split_ops(O.Oracle(n, 0.1, lam=500.0), U)
    for a, b in zip(out, U):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("sigma", [0.25, 0.6])
def test_filter_single_mode_symbol(sigma):
    """Each mode of q and W is multiplied by 1 - sigma sin^4(theta/2); h and K
    are untouched; a constant passes (theta = 0)."""
    n = 64
    x = np.arange(n)
    for j in (1, 5, 16, 23, 32):
        th = 2 * np.pi * j / n
        base = [np.full(n, 1.0), np.full(n, 0.3), np.full(n, 1.0), np.full(n, -0.2)]
        mode = np.cos(th * x + 0.4)
        U = [base[0] + 0.01 * mode, base[1] + 0.05 * mode, base[2] + 0.02 * mode, base[3] + 0.04 * mode]
        o = O.Oracle(n, 0.1, lam=500.0, filter_sigma=sigma)
        out = _split_ops(o, U)
        F = 1.0 - sigma * math.sin(th / 2) ** 4
        assert np.array_equal(out[0], U[0]) and np.array_equal(out[2], U[2])
        assert np.max(np.abs(out[1] - (base[1] + F * 0.05 * mode))) < 1e-15, j
        assert np.max(np.abs(out[3] - (base[3] + F * 0.04 * mode))) < 1e-15, j


def test_filter_mask_selects_fields():
    n = 32
    U = _smooth_state(n, 2)
    U[0] = U[0] + 0.01 * (-1.0) ** np.arange(n)       # grid-scale content in every field
    U[2] = U[2] + 0.01 * (-1.0) ** np.arange(n)
    out = _split_ops(O.Oracle(n, 0.1, lam=500.0, filter_sigma=0.25, filter_mask=0b0101), U)
    assert not np.array_equal(out[0], U[0]) and not np.array_equal(out[2], U[2])
    assert np.array_equal(out[1], U[1]) and np.array_equal(out[3], U[3])


@pytest.mark.parametrize("bc", ["wall", "transmissive"])
def test_filter_physical_ends(bc):
    """Wall: equals the periodic filter of the mirror-doubled domain (q odd, W
    even).  Transmissive: equals the periodic filter of a domain padded with
    copies of the end cells (zero-order extrapolation, A10)."""
    n = 40
    rng = np.random.default_rng(5)
    U = [1 + 0.05 * rng.standard_normal(n), 0.1 * rng.standard_normal(n),
         1 + 0.05 * rng.standard_normal(n), 0.05 * rng.standard_normal(n)]
    out = _split_ops(O.Oracle(n, 0.1, lam=300.0, bc=(bc, bc), filter_sigma=0.25), U)
    if bc == "wall":
        dbl = [np.concatenate([f, s * f[::-1]]) for f, s in zip(U, (1, -1, 1, 1))]
        ref = _split_ops(O.Oracle(2 * n, 0.1, lam=300.0, filter_sigma=0.25), dbl)
        for k in (1, 3):
            assert np.max(np.abs(out[k] - ref[k][:n])) < 1e-16
    else:
        pad = 4
        ext = [np.concatenate([np.full(pad, f[0]), f, np.full(pad, f[-1])]) for f in U]
        ref = _split_ops(O.Oracle(n + 2 * pad, 0.1, lam=300.0, filter_sigma=0.25), ext)
        for k in (1, 3):
            # interior cells use no ghost; cells 0,1 and n-2,n-1 see copies
            assert np.max(np.abs(out[k] - ref[k][pad:pad + n])) < 1e-16


@pytest.mark.parametrize("order", [2, 1])
def test_filtered_step_matches_filtered_symbol(order):
    """One filtered SI step on a single mode about rest equals the filtered
    4x4 symbol (LT.step_symbol with filter_sigma) to O(eps)."""
    n, dx, h0, lam, sigma = 64, 0.2, 1.0, 500.0, 0.25
    dt = 2.7 * dx / math.sqrt(G * h0 + lam / 3)
    x = np.arange(n)
    eps = 1e-8
    o = O.Oracle(n, dx, lam=lam, order=order, filter_sigma=sigma)
    for k in (3, 11, 22, 29):
        th = 2 * np.pi * k / n
        Gm = LT.step_symbol(th, dx, h0, lam, G, dt, order=order, filter_sigma=sigma)
        Gu = LT.step_symbol(th, dx, h0, lam, G, dt, order=order)
        assert np.max(np.abs(Gm - Gu)) > 1e-3        # the filter is visible at this theta
        for j in range(4):
            v = np.zeros(4)
            v[j] = 1.0
            pert = eps * np.outer(v, np.cos(th * x))
            U2 = o.step([h0 + pert[0], pert[1], h0 * h0 + pert[2], pert[3]], dt)
            resp = np.array([U2[0] - h0, U2[1], U2[2] - h0 * h0, U2[3]])
            pred = eps * np.real(np.outer(Gm[:, j], np.exp(1j * th * x)))
            scale = np.max(np.abs(pred)) + eps * 1e-3
            assert np.max(np.abs(resp - pred)) <= 2e-5 * scale + 1e-15, (k, j)


# --------------------------------------------------------------------------
# A10 relaxation zones (A10)
# --------------------------------------------------------------------------
def _relax_params():
    h0 = 0.4
    omega = 2 * math.pi / 2.02
    k = 1.6812
    return dict(x_min=0.0, level=h0, gen_x1=4.0, gen_rate=0.1, amp=0.01, omega=omega, k=k,
                cp=omega / k, sp_x0=30.0, sp_rate=0.1)


def test_relaxation_one_application():
    """U - s(x)(U - target(x, t)), written from DESIGN.md A10: generation zone
    [x_min, x_min + 4] with s = rate (1 - (x - x_min)/4)^2 towards eta = a sin(omega t
    - k (x - x_min)), h = level + eta - b, u = c_p eta/level, K = h (h + 1.5 b), W = 0;
    sponge [30, 40] with s = rate ((x - 30)/10)^2 towards the lake at rest."""
    n, L = 400, 40.0
    dx = L / n
    xc = (np.arange(n) + 0.5) * dx
    rng = np.random.default_rng(9)
    b = 0.05 * np.sin(xc / 3.0)
    rp = _relax_params()
    h = 0.4 - b + 0.01 * rng.standard_normal(n)
    U = [h, 0.01 * rng.standard_normal(n), h * (h + 1.5 * b) + 1e-3 * rng.standard_normal(n),
         0.01 * rng.standard_normal(n)]
    t = 1.37
    o = O.Oracle(n, dx, lam=1000.0, bc=("transmissive", "transmissive"), b=b, relax=rp)
    out = _split_ops(o, U, t=t)
    # the dt = 0 stage maps K -> (K - 1.5 h b) + 1.5 h b: a few ulp off K with b != 0
    Kst = (U[2] - 1.5 * U[0] * b) + 1.5 * U[0] * b
    s = np.zeros(n)
    tgt = [np.zeros(n) for _ in range(4)]
    gen = xc <= 4.0
    r = 1.0 - xc[gen] / 4.0
    s[gen] = 0.1 * r * r
    eta = 0.01 * np.sin(rp["omega"] * t - rp["k"] * xc[gen])
    th = 0.4 + eta - b[gen]
    tgt[0][gen] = th
    tgt[1][gen] = th * (rp["cp"] * eta / 0.4)
    tgt[2][gen] = th * (th + 1.5 * b[gen])
    sp = xc >= 30.0
    r = (xc[sp] - 30.0) / 10.0
    s[sp] = 0.1 * r * r
    th = 0.4 - b[sp]
    tgt[0][sp] = th
    tgt[2][sp] = th * (th + 1.5 * b[sp])
    for kf, f in enumerate([U[0], U[1], Kst, U[3]]):
        ref = f - s * (f - tgt[kf])
        assert np.max(np.abs(out[kf] - ref)) < 1e-15, kf
    assert np.array_equal(out[1][~(gen | sp)], U[1][~(gen | sp)])   # outside the zones: untouched


def test_wavemaker_target_is_a_right_going_linear_wave():
    """With rate 1 the first cell relaxes onto the target; along the zone the
    target's q/h is c_p times eta/h0 and its phase travels right at omega/k."""
    n, L = 4000, 40.0
    dx = L / n
    rp = _relax_params()
    rp.update(gen_rate=1.0, sp_rate=0.0)
    o = O.Oracle(n, dx, lam=1000.0, bc=("transmissive", "transmissive"), relax=rp)
    h = np.full(n, 0.4)
    z = np.zeros(n)
    cell = 0                                      # s = (1 - dx/(2*4))^2 ~ 1
    vals = []
    for t in np.linspace(0.0, 2.02, 9):
        out = _split_ops(o, [h, z, h * h, z], t=t)
        r = 1.0 - (cell + 0.5) * dx / 4.0
        s = r * r
        eta = (out[0][cell] - 0.4) / s               # target eta at this cell
        u = out[1][cell] / s / (0.4 + eta)
        vals.append((t, eta, u))
    for t, eta, u in vals:
        assert abs(u - (rp["omega"] / rp["k"]) * eta / 0.4) < 1e-14
        assert abs(eta - 0.01 * math.sin(rp["omega"] * t - rp["k"] * 0.5 * dx)) < 1e-12


# --------------------------------------------------------------------------
# A24 Picard fixed point = the un-frozen depth equation solved by Newton
# --------------------------------------------------------------------------
def _unfrozen_residual(hb, h, tau, dx, lam, g, periodic):
    """P:500-512 (reading A1) with beta1, beta2 (hence beta = kappa and delta)
    evaluated at the unknown hbar (P:279-285 un-frozen), a^2 and alpha at E
    (P:142-143), on a state with u = 0, eta = h, w = 0: fluxes vanish, so
    q^dag = 0, W^dag = lam tau, H^dag = h^2 + tau W^dag = h^2 + lam tau^2."""
    n = len(h)
    Hd = h * h + lam * tau * tau
    sg = 1.0                                       # eta/h at E
    alpha = -(2 * sg - 1) / (3 * h)
    a2 = g * h + (lam / 3) * sg * (3 * sg - 1)
    beta1 = 1 + lam * tau * tau / (hb * hb)          # P:505 at hbar
    beta2 = 2 * lam * tau * tau / (beta1 * beta1 * hb ** 3)   # P:506 at hbar
    beta = a2 + lam * alpha * beta2 * Hd
    delta = alpha / beta1
    if periodic:
        nb = lambda a, s: np.roll(a, -s)
    else:
        def nb(a, s):                                # mirror ghosts (A10)
            out = np.roll(a, -s)
            if s == 1:
                out[-1] = a[-1]
            else:
                out[0] = a[0]
            return out
    t2 = tau * tau / (dx * dx)
    rr = t2 * (beta + nb(beta, 1)) / 2
    rl = t2 * (nb(beta, -1) + beta) / 2
    mr = lam * tau * tau / (2 * dx * dx) * (delta + nb(delta, 1))
    ml = lam * tau * tau / (2 * dx * dx) * (nb(delta, -1) + delta)
    if not periodic:
        rl[0] = rr[-1] = 0.0
    rhs = h + mr * (nb(Hd, 1) - Hd) - ml * (Hd - nb(Hd, -1))     # q^dag = 0
    lhs = hb * (1 + rl + rr) - rr * nb(hb, 1) - rl * nb(hb, -1)
    return lhs - rhs, beta, delta, Hd


def _newton(h, tau, dx, lam, g, periodic):
    hb = h.copy()
    for _ in range(30):
        F = _unfrozen_residual(hb, h, tau, dx, lam, g, periodic)[0]
        J = np.empty((len(h), len(h)))
        for j in range(len(h)):
            e = np.zeros(len(h))
            e[j] = 1e-7
            J[:, j] = (_unfrozen_residual(hb + e, h, tau, dx, lam, g, periodic)[0]
                       - _unfrozen_residual(hb - e, h, tau, dx, lam, g, periodic)[0]) / 2e-7
        d = np.linalg.solve(J, -F)
        hb = hb + d
        if np.max(np.abs(d)) < 1e-15:
            break
    return hb


@pytest.mark.parametrize("bc", ["periodic", "wall"])
@pytest.mark.parametrize("lam", [300.0, 5000.0])
def test_picard_fixed_point_solves_unfrozen_equation(bc, lam):
    n, dx = 8, 0.15
    rng = np.random.default_rng(13)
    h = 1.0 + 0.25 * np.cos(2 * np.pi * np.arange(n) / n + 0.3) + 0.05 * rng.standard_normal(n)
    if bc == "wall":
        h = 1.0 + 0.2 * np.cos(np.pi * (np.arange(n) + 0.5) / n) + 0.03 * rng.standard_normal(n)
    z = np.zeros(n)
    U = [h, z, h * h, z]
    tau = 2.5 * dx / math.sqrt(G * 1.3 + lam / 3)
    hb = _newton(h, tau, dx, lam, G, bc == "periodic")
    F, beta, delta, Hd = _unfrozen_residual(hb, h, tau, dx, lam, G, bc == "periodic")
    assert np.max(np.abs(F)) < 1e-14
    out, _ = O.Oracle(n, dx, lam=lam, bc=(bc, bc), picard=40).stage(U, U, tau)
    lin, _ = O.Oracle(n, dx, lam=lam, bc=(bc, bc), picard=0).stage(U, U, tau)
    assert np.max(np.abs(lin[0] - hb)) > 1e-9          # the frozen stage differs
    assert np.max(np.abs(out[0] - hb)) < 1e-13, np.max(np.abs(out[0] - hb))
    # back-substitution from the Newton depth: qbar, Hbar, Wbar
    if bc == "periodic":
        hr, hl = np.roll(hb, -1), np.roll(hb, 1)
        Hr, Hl = np.roll(Hd, -1), np.roll(Hd, 1)
    else:
        hr, hl = np.append(hb[1:], hb[-1]), np.insert(hb[:-1], 0, hb[0])
        Hr, Hl = np.append(Hd[1:], Hd[-1]), np.insert(Hd[:-1], 0, Hd[0])
    qb = -(tau / (2 * dx)) * beta * (hr - hl) - (lam * tau / (2 * dx)) * delta * (Hr - Hl)
    Hb = Hd / (1 + lam * tau * tau / hb ** 2)
    Wb = lam * tau - lam * tau * Hb / hb ** 2
    assert np.max(np.abs(out[1] - qb)) < 1e-11
    assert np.max(np.abs(out[2] - Hb)) < 1e-13
    assert np.max(np.abs(out[3] - Wb)) < 1e-10 * lam * tau
