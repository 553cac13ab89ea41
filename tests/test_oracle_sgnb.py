"""Pins of the oracle's bathymetric classical SGN scheme (reading
A26) against what the paper and the mathematics fix.

  * b = 0 reproduces the flat scheme bit for bit
  * the closure (kappa, rho, Q of P:570-578) is checked against the PRIMITIVE
    mild-slope model of P:175-186 (momentum with p~_nh), solved spectrally for
    phi := Du/Dt + g zeta_x on a periodic grid: the oracle's right-hand side
    converges to it at O(dx^2) -- a wrong sign or factor in kappa, rho or Q,
    or a missing g h b_x, breaks the convergence
  * lake at rest: phi = 0 exactly, the spurious tendency is O(dx^2)
  * mass conservation (flux form), periodic and walls
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W

G = 9.81


def _fx(f, L):
    k = 2 * np.pi * np.fft.fftfreq(len(f), d=L / len(f))
    return np.real(np.fft.ifft(1j * k * np.fft.fft(f)))


def _primitive_rhs(h, q, b, L):
    """(h_t, (hu)_t) of P:175-186 on a periodic grid, spectral derivatives:
    h Du/Dt + g h zeta_x = -(h p~)_x - 3/2 p~ b_x,
    p~ = -(h^2/3)(Du/Dt)_x + (h b_x/2) Du/Dt + (2/3) h^2 u_x^2 + h^2 u^2 b_xx.
    With a := Du/Dt the equation is linear in a; solved densely."""
    n = len(h)
    u = q / h
    zeta = h + b
    ux, bx, zx = _fx(u, L), _fx(b, L), _fx(zeta, L)
    bxx = _fx(bx, L)

    def ptil(a):
        return -(h * h / 3.0) * _fx(a, L) + (h * bx / 2.0) * a + (2.0 / 3.0) * h * h * ux * ux + h * h * u * u * bxx

    def resid(a):             # h a + g h zeta_x + (h p~)_x + 1.5 p~ b_x
        p = ptil(a)
        return h * a + G * h * zx + _fx(h * p, L) + 1.5 * p * bx

    r0 = resid(np.zeros(n))
    M = np.empty((n, n))
    for j in range(n):
        e = np.zeros(n)
        e[j] = 1.0
        M[:, j] = resid(e) - r0
    a = np.linalg.solve(M, -r0)
    ht = -_fx(q, L)
    qt = h * (a - u * ux) + u * ht      # (hu)_t = h u_t + u h_t, u_t = Du/Dt - u u_x
    return ht, qt


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_sgnb_zero_bathymetry_is_the_flat_scheme(bc):
    w = W.random_smooth(300, 1, seed=5, amp=0.08, bc=(bc, bc))
    U = w.state(0)
    a = O.Oracle(w.n, w.dx, bc=w.bc).sgn_step(U, 0.01)
    b = O.Oracle(w.n, w.dx, bc=w.bc, b=np.zeros(w.n)).sgn_step(U, 0.01)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_sgnb_rhs_converges_to_the_primitive_mild_slope_model():
    L = 20.0
    kx = 2 * np.pi / L
    errs = []
    for n in (96, 192, 384):
        x = W.cell_centres(0.0, L, n)
        b = 0.15 * np.sin(kx * x + 0.4) + 0.1 * np.cos(3 * kx * x)     # |b_x| up to ~0.14
        h = 1.0 + 0.1 * np.cos(kx * x) - b
        q = h * (0.2 + 0.15 * np.sin(kx * x))
        ht, qt = _primitive_rhs(h, q, b, L)
        o = O.Oracle(n, L / n, b=b)
        Lh, Lq = o.sgn_rhs(h, q)
        errs.append([np.max(np.abs(Lh - ht)) / np.max(np.abs(ht)), np.max(np.abs(Lq - qt)) / np.max(np.abs(qt))])
    errs = np.array(errs)
    orders = np.log2(errs[:-1] / errs[1:])
    assert np.all(errs[-1] < 5e-3), errs
    assert np.all(orders > 1.7), (errs, orders)


def test_sgnb_lake_at_rest_second_order():
    """zeta = const, u = 0: phi = 0 exactly (every right-hand side term of the
    phi equation vanishes); the shallow-water part leaves an O(dx^2) tendency."""
    L = 20.0
    res = []
    for n in (100, 200, 400):
        x = W.cell_centres(0.0, L, n)
        b = 0.2 * np.sin(2 * np.pi * x / L)
        h = 1.0 - b
        Lh, Lq = O.Oracle(n, L / n, b=b).sgn_rhs(h, np.zeros(n))
        res.append(max(np.max(np.abs(Lh)), np.max(np.abs(Lq))))
    orders = np.log2(np.array(res[:-1]) / np.array(res[1:]))
    assert np.all(orders > 1.8), (res, orders)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_sgnb_mass_conservation(bc):
    w = W.random_smooth(400, 1, seed=9, amp=0.05, bc=(bc, bc), bathy=0.05)
    o = O.Oracle(w.n, w.dx, bc=w.bc, b=w.b)
    U = w.state(0)
    m0 = np.sum(U[0])
    U2, t, s = o.sgn_run(U, cfl=0.9, steps=100)
    assert abs(np.sum(U2[0]) - m0) <= 1e-13 * m0
