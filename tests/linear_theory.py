"""Closed-form linear theory used as PINS of the oracle (not an implementation).

Everything here is derived by hand from the paper's equations, linearised about
flat rest (h0, u = 0, eta = h0, w = 0), and is written in Fourier space -- a
different representation from the oracle's cell loops, so that a dropped term,
a wrong sign, a wrong index or a transposed operand in the oracle shows up as a
mismatch.  Derivations: DESIGN.md section 4 (and SURVEY.md App. A.2, A.5).

Stage symbol (linearisation of P:502-515 under readings A1, A4, A5):
  at rest F^q = q^2/h and F^W = qW/h have no linear part and F^H = qH/h has the
  linear part h0 q'; Rusanov's alpha = |u| is O(eps) so its dissipation is
  quadratic; the coefficient perturbations multiply background differences that
  vanish at rest, so only their background values enter:
    b1 = h0^2/(h0^2 + lam tau^2),  beta0 = g h0 + (2 lam/3) b1,
    delta0 = -b1/(3 h0),  k2 = 2 lam tau^2 h0/(h0^2 + lam tau^2)
  and with D = i sin(th)/dx (wide centred difference),
  C = -4 sin^2(th/2)/dx^2 (compact second difference),
  M = MUSCL face-average flux difference:
    H' = H'_R + tau W'_R - tau h0 M q'_E
    q' = q'_R
    hbar' = (h'_R - tau D q' + lam tau^2 delta0 C H') / (1 - tau^2 beta0 C)
    qbar' = q' - tau beta0 D hbar' - lam tau delta0 D H'
    Hbar' = b1 H' + k2 hbar'                                    (P:514 linearised)
    Wbar' = W'_R - (lam tau/h0^2) Hbar' + (2 lam tau/h0) hbar'  (P:515 linearised)
Step: IMEX efficient form.
"""
from __future__ import annotations

import numpy as np

GAMMA = 1.0 - 1.0 / np.sqrt(2.0)
C_E = 1.0 / (2.0 * GAMMA)


def stage_symbol(theta, dx, h0, lam, g, tau, order=2):
    """Return S(E', R') -> U' (4-vectors over (h, q, H, W)) for one Fourier mode."""
    e = np.exp(1j * theta)
    D = 1j * np.sin(theta) / dx
    Cc = -4.0 * np.sin(theta / 2.0) ** 2 / dx ** 2
    if order == 2:
        face = (1 + e) / 2 + (e - 1 / e - e ** 2 + 1) / 8
    else:
        face = (1 + e) / 2
    M = (1 - 1 / e) * face / dx
    b1 = h0 ** 2 / (h0 ** 2 + lam * tau ** 2)
    beta0 = g * h0 + 2.0 * lam / 3.0 * b1
    delta0 = -b1 / (3.0 * h0)
    k2 = 2.0 * lam * tau ** 2 * h0 / (h0 ** 2 + lam * tau ** 2)

    def S(Ev, Rv):
        hR, qR, HR, WR = Rv
        Hd = HR + tau * WR - tau * h0 * M * Ev[1]
        qd = qR
        hb = (hR - tau * D * qd + lam * tau ** 2 * delta0 * Cc * Hd) / (1 - tau ** 2 * beta0 * Cc)
        qb = qd - tau * beta0 * D * hb - lam * tau * delta0 * D * Hd
        Hb = b1 * Hd + k2 * hb
        Wb = WR - lam * tau / h0 ** 2 * Hb + 2 * lam * tau / h0 * hb
        return np.array([hb, qb, Hb, Wb])

    return S


def step_symbol(theta, dx, h0, lam, g, dt, order=2, stages=2, filter_sigma=0.0):
    """4x4 amplification matrix of one SI-IMEX step about rest."""
    G = np.zeros((4, 4), complex)
    if stages == 2:
        wE = C_E / GAMMA
        wR = (1 - GAMMA) / GAMMA
        S = stage_symbol(theta, dx, h0, lam, g, GAMMA * dt, order)
    else:
        S = stage_symbol(theta, dx, h0, lam, g, dt, order)
    for k in range(4):
        U = np.zeros(4, complex)
        U[k] = 1.0
        U1 = S(U, U)
        if stages == 2:
            E2 = (1 - wE) * U + wE * U1
            R2 = (1 - wR) * U + wR * U1
            G[:, k] = S(E2, R2)
        else:
            G[:, k] = U1
    if filter_sigma > 0:
        # A19: f <- f - (sigma/16) d4 f on q and W; d4 symbol = 16 sin^4(theta/2)
        F = 1.0 - filter_sigma * np.sin(theta / 2.0) ** 4
        G[1, :] *= F
        G[3, :] *= F
    return G


def max_growth(dx, h0, lam, g, dt, order=2, stages=2, filter_sigma=0.0, thetas=None):
    """max over theta of the spectral radius of step_symbol."""
    if thetas is None:
        thetas = np.linspace(1e-3, np.pi, 600)
    best = 0.0
    for th in thetas:
        r = np.max(np.abs(np.linalg.eigvals(step_symbol(th, dx, h0, lam, g, dt, order, stages,
                                                        filter_sigma))))
        best = max(best, r)
    return best


def hsgn_slow_omega(k, h0, lam, g):
    """Slow branch of the linear hSGN dispersion relation, derived from P:101-111
    about rest:  p' = (g h0 + lam/3) h' - (lam/3) eta',  eta'_t = w',
    h0 w'_t = -(lam/h0)(eta' - h')  =>
    h0^2 W^2 - [lam (1 + (k h0)^2/3) + g h0^3 k^2] W + lam g h0 k^2 = 0, W = omega^2."""
    a = h0 ** 2
    b = -(lam * (1 + (k * h0) ** 2 / 3.0) + g * h0 ** 3 * k ** 2)
    c = lam * g * h0 * k ** 2
    disc = np.sqrt(b * b - 4 * a * c)
    Wslow = (-b - disc) / (2 * a)
    return np.sqrt(Wslow)


def sgn_omega(k, h0, g):
    """SGN dispersion omega^2 = g h0 k^2 / (1 + (k h0)^2/3) (limit lam -> inf)."""
    return np.sqrt(g * h0 * k * k / (1 + (k * h0) ** 2 / 3.0))


def slow_mode_state(x, k, eps, h0, lam, g, t=0.0):
    """Primitive perturbation of the slow eigenmode (derived above):
    h' = eps cos(phi), u' = (omega/(k h0)) h', eta' = lam h'/(lam - omega^2 h0^2),
    w' = eta'_t; phi = k x - omega t."""
    om = hsgn_slow_omega(k, h0, lam, g)
    phi = k * x - om * t
    hp = eps * np.cos(phi)
    up = om / (k * h0) * hp
    eta_hat = lam / (lam - om * om * h0 * h0) if lam > 0 else 1.0
    etap = eta_hat * hp
    wp = eta_hat * eps * om * np.sin(phi)
    h = h0 + hp
    eta = h0 + etap
    return h, h * up, h * eta, h * wp


def explicit_symbol(theta, dx, h0, lam, g, dt, order=2, stages=2, filter_sigma=0.0):
    """4x4 amplification matrix of one explicit step (Heun P:480)
    about rest.  Linearising L(U): the convective fluxes q u and W u are
    quadratic and Rusanov's alpha = |u| is O(eps), so only F^H = H q / h keeps
    the linear part h0 q' (through the MUSCL face average M); at rest
    sigma = 1, alpha0 = -1/(3 h0) and a0^2 = g h0 + (lam/3) - lam h0 alpha0
    = g h0 + 2 lam/3; lam (H/h^2 - 1) linearises to
    (lam/h0^2)(H' - 2 h0 h').  With D = i sin(th)/dx:
      L_h = -D q'
      L_q = -a0^2 D h' - lam alpha0 D H'
      L_H = -h0 M q' + W'
      L_W = (2 lam/h0) h' - (lam/h0^2) H'
    Euler: G = I + dt A; Heun: G = I + dt A + (dt A)^2 / 2."""
    e = np.exp(1j * theta)
    D = 1j * np.sin(theta) / dx
    if order == 2:
        face = (1 + e) / 2 + (e - 1 / e - e ** 2 + 1) / 8
    else:
        face = (1 + e) / 2
    M = (1 - 1 / e) * face / dx
    a2 = g * h0 + 2.0 * lam / 3.0
    al = -1.0 / (3.0 * h0)
    A = np.array([[0, -D, 0, 0],
                  [-a2 * D, 0, -lam * al * D, 0],
                  [0, -h0 * M, 0, 1.0],
                  [2 * lam / h0, 0, -lam / h0 ** 2, 0]], dtype=complex)
    I = np.eye(4, dtype=complex)
    G = I + dt * A if stages == 1 else I + dt * A + 0.5 * (dt * A) @ (dt * A)
    if filter_sigma > 0:
        F = 1.0 - filter_sigma * np.sin(theta / 2.0) ** 4
        G[1, :] *= F
        G[3, :] *= F
    return G


def explicit_max_growth(dx, h0, lam, g, dt, order=2, stages=2, filter_sigma=0.0, thetas=None):
    if thetas is None:
        thetas = np.linspace(1e-3, np.pi, 600)
    return max(np.max(np.abs(np.linalg.eigvals(explicit_symbol(th, dx, h0, lam, g, dt, order, stages,
                                                               filter_sigma)))) for th in thetas)


def sgn_symbol(theta, dx, h0, g, dt, order=2, stages=2):
    """2x2 amplification matrix over (h, q) of one step of the classical SGN
    scheme (reading A23) about rest.  Shallow-water part: Rusanov
    on MUSCL faces with alpha = sqrt(g h0) at rest (linear dissipation), flux
    Jacobian [[0, 1], [g h0, 0]]; face-state symbols sm = 1 + (e - 1/e)/4,
    sp = e - (e^2 - 1)/4 (order 1: 1, e).  phi: h0 phi - (h0^3/(3 dx^2)) d2 phi
    = h*, h* = -(g h0^3/(6 dx^3)) [(e^2 - 2e + 1) - (1 - 2/e + 1/e^2)] h'
    (the (u_x)^2 terms are quadratic).  L = (-(1 - 1/e)/dx Fh, -(1 - 1/e)/dx Fq
    + h0 phi)."""
    e = np.exp(1j * theta)
    if order == 2:
        sm = 1 + (e - 1 / e) / 4
        sp = e - (e * e - 1) / 4
    else:
        sm, sp = 1.0, e
    c0 = np.sqrt(g * h0)
    J = np.array([[0, 1], [g * h0, 0]], dtype=complex)
    F = 0.5 * J * (sm + sp) - 0.5 * c0 * (sp - sm) * np.eye(2)
    D = (1 - 1 / e) / dx
    hstar = -(g * h0 ** 3 / (6 * dx ** 3)) * ((e * e - 2 * e + 1) - (1 - 2 / e + 1 / (e * e)))
    phi = hstar / (h0 - (h0 ** 3 / (3 * dx * dx)) * (e - 2 + 1 / e))
    A = -D * F
    A[1, 0] += h0 * phi
    I = np.eye(2, dtype=complex)
    return I + dt * A if stages == 1 else I + dt * A + 0.5 * (dt * A) @ (dt * A)
