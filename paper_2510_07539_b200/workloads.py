"""Seeded synthetic inputs for the SI-IMEX hSGN hot path.

This module holds ONLY input generators (initial states, bathymetry, per-member
parameters) and closed-form reference profiles.  It contains none of the SI
method's arithmetic, and it is the one module shared by the oracle tests and the
CUDA path (DESIGN.md section 5 gives the recipe of each config).

Every generator returns fp64 numpy arrays (h, q, K, W) in the state convention
of DESIGN.md: q = h u, K = h eta (flat) or h (eta + 3 b / 2),
W = h w.

Closed forms followed:
  * SGN solitary wave: h = h0 (1 + eps sech^2(kappa (x - x0))),
    u = C (1 - h0/h), C = sqrt(g h0 (1 + eps)), kappa = sqrt(3 eps / (4 h0^2 (1 + eps))),
    eta = h, w = -h u_x (A11: K = h^2, W = -h^2 u_x, u_x analytic).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

G_DEFAULT = 9.81  # P:646 (A14: m/s^2)


@dataclass
class Workload:
    name: str
    n: int                      # cells per member
    members: int
    x_min: float
    x_max: float
    bc: tuple                   # ("periodic","periodic") | ("wall","wall") | ...
    lam: np.ndarray             # [members]
    h: np.ndarray               # [members, n] (or [n] flattened as [1, n])
    q: np.ndarray
    K: np.ndarray
    W: np.ndarray
    b: np.ndarray | None = None  # [n] shared by all members, or None
    g: float = G_DEFAULT
    cfl: float = 2.0
    mcfl: float = 0.5
    steps: int | None = None
    t_end: float | None = None
    filter_sigma: float = 0.0
    meta: dict = field(default_factory=dict)

    @property
    def dx(self) -> float:
        return (self.x_max - self.x_min) / self.n

    def x(self) -> np.ndarray:
        return cell_centres(self.x_min, self.x_max, self.n)

    def state(self, m: int = 0):
        return [self.h[m], self.q[m], self.K[m], self.W[m]]

    def subset(self, members) -> "Workload":
        idx = np.asarray(members)
        return Workload(self.name, self.n, len(idx), self.x_min, self.x_max, self.bc,
                        self.lam[idx].copy(), self.h[idx].copy(), self.q[idx].copy(),
                        self.K[idx].copy(), self.W[idx].copy(), self.b, self.g, self.cfl,
                        self.mcfl, self.steps, self.t_end, self.filter_sigma, dict(self.meta))


def cell_centres(x_min: float, x_max: float, n: int) -> np.ndarray:
    """x_i = x_min + (i + 1/2) dx."""
    dx = (x_max - x_min) / n
    return x_min + (np.arange(n, dtype=np.float64) + 0.5) * dx


def _wrap(d: np.ndarray, L: float | None) -> np.ndarray:
    if L is None:
        return d
    return d - L * np.floor(d / L + 0.5)  # minimum image in [-L/2, L/2)


def soliton_params(h0: float, A: float, g: float = G_DEFAULT):
    """(eps, kappa, C) of the SGN solitary wave."""
    eps = A / h0
    kappa = math.sqrt(3.0 * eps / (4.0 * h0 * h0 * (1.0 + eps)))
    C = math.sqrt(g * h0 * (1.0 + eps))
    return eps, kappa, C


def soliton_exact(x, t, h0, A, x0, g=G_DEFAULT, L=None):
    """Exact SGN soliton translated by C t (A13): returns (h, u)."""
    eps, kappa, C = soliton_params(h0, A, g)
    d = _wrap(np.asarray(x, dtype=np.float64) - x0 - C * t, L)
    s2 = 1.0 / np.cosh(kappa * d) ** 2
    h = h0 * (1.0 + eps * s2)
    u = C * (1.0 - h0 / h)
    return h, u


def soliton_state(x, h0, A, x0, g=G_DEFAULT, L=None):
    """hSGN state of the SGN soliton with eta = h, w = -h u_x (A11)."""
    eps, kappa, C = soliton_params(h0, A, g)
    d = _wrap(np.asarray(x, dtype=np.float64) - x0, L)
    th = np.tanh(kappa * d)
    s2 = 1.0 / np.cosh(kappa * d) ** 2
    h = h0 * (1.0 + eps * s2)
    hx = -2.0 * h0 * eps * kappa * s2 * th
    u = C * (1.0 - h0 / h)
    ux = C * h0 * hx / (h * h)
    return h, h * u, h * h, -h * h * ux


def multi_soliton_state(x, amps, pos, g=G_DEFAULT, L=None, h0=1.0):
    """Superposed solitary waves (cfg3): h = h0 + sum_j A_j sech^2(kappa_j d_j),
    u = sum_j C_j (1 - h0 / (h0 + A_j sech^2)), eta = h, w = -h u_x (analytic)."""
    h = np.full_like(x, h0)
    u = np.zeros_like(x)
    ux = np.zeros_like(x)
    for A, x0 in zip(amps, pos):
        _, kappa, C = soliton_params(h0, A, g)
        d = _wrap(x - x0, L)
        th = np.tanh(kappa * d)
        s2 = 1.0 / np.cosh(kappa * d) ** 2
        hj = h0 + A * s2
        hjx = -2.0 * A * kappa * s2 * th
        h = h + A * s2
        u = u + C * (1.0 - h0 / hj)
        ux = ux + C * h0 * hjx / (hj * hj)
    return h, h * u, h * h, -h * h * ux


# --------------------------------------------------------------------------
# BASELINE.json configs (synthetic stand-ins)
# --------------------------------------------------------------------------

def cfg1(n: int = 1000, lam: float = 500.0, x0: float = -50.0) -> Workload:
    """Solitary wave, periodic [-100, 100), h0 = 1, a = 0.2, lambda = 500, t_end = 20;
    dt = min(2.7 dx / nu_max, 0.5 dx / u_max) (A12); A19 filter on (seeded-rest
    pin decides it, A19)."""
    x = cell_centres(-100.0, 100.0, n)
    h, q, K, W = soliton_state(x, 1.0, 0.2, x0, L=200.0)
    return Workload("cfg1_soliton", n, 1, -100.0, 100.0, ("periodic", "periodic"),
                    np.array([lam]), h[None], q[None], K[None], W[None], cfl=2.7, mcfl=0.5,
                    t_end=20.0, filter_sigma=0.25, meta=dict(h0=1.0, A=0.2, x0=x0, L=200.0))


def cfg2(lam: float, n: int = 1 << 16, width_cells: float = 50.0) -> Workload:
    """Dispersive dam break on [-300, 300] with walls: h = 1.8 left / 1.0 right,
    u = 0, K = h^2, W = 0, t_end = 48.  The step is regularised as a tanh over
    width_cells cells (50 by default, ~0.46 m at N = 2^16): the unlimited MUSCL
    of the paper breaks down (coercivity) within ~50 steps on a sharp
    step at every lambda and on a 5-cell tanh at lambda >= 1e3 (A20);
    width_cells = 0 gives the sharp step."""
    x = cell_centres(-300.0, 300.0, n)
    dx = 600.0 / n
    if width_cells > 0:
        h = 1.4 - 0.4 * np.tanh(x / (width_cells * dx))
    else:
        h = np.where(x < 0.0, 1.8, 1.0)
    z = np.zeros_like(h)
    return Workload(f"cfg2_dambreak_lam{lam:g}", n, 1, -300.0, 300.0, ("wall", "wall"),
                    np.array([lam]), h[None], z[None].copy(), (h * h)[None], z[None].copy(),
                    cfl=2.0, mcfl=0.5, t_end=48.0, filter_sigma=0.25)


def cfg2_lambdas(lams=(1e2, 1e3, 1e4), n: int = 1 << 16, width_cells: float = 50.0) -> Workload:
    """cfg2's lambda values as the members of one ensemble (same initial dam break;
    each member its own dt and t_end clipping): the three runs in one context."""
    one = cfg2(lams[0], n, width_cells)
    k = len(lams)
    rep = lambda a: np.repeat(a, k, axis=0)
    return Workload("cfg2_dambreak_lambdas", n, k, one.x_min, one.x_max, one.bc, np.array(lams, dtype=float),
                    rep(one.h), rep(one.q), rep(one.K), rep(one.W), cfl=one.cfl, mcfl=one.mcfl,
                    t_end=one.t_end, filter_sigma=one.filter_sigma)


def cfg3(members: int = 4096, n: int = 4096, seed: int = 7539003, dx: float = 0.1,
         first_member: int = 0, filter_sigma: float = 0.25) -> Workload:
    """Batched ensemble: `members` periodic domains of n cells (dx = 0.1); per member
    1-3 solitary waves with amplitudes U(0.05, 0.3), positions U[0, L), and
    lambda = 10^U(2, 4); 200 steps at CFL_IMEX = 2, MCFL = 0.5.  A19 filter on by
    default: the literal scheme amplifies a 1e-14 perturbation to 1e-4 within the
    200 steps in some members (A19), so no full-run parity is possible
    without it; filter_sigma = 0 gives the literal scheme.

    Each member m draws from its own PCG64 stream seeded with (seed, m), in the
    order n_s, amplitudes[3], positions[3], lambda, so member m's state does not
    depend on how many members are generated or which shard does it: any subset
    [first_member, first_member + members) equals the same rows of the full
    ensemble."""
    L = n * dx
    x = cell_centres(0.0, L, n)
    H = np.empty((members, n)); Q = np.empty((members, n))
    KK = np.empty((members, n)); WW = np.empty((members, n))
    lam = np.empty(members)
    for mi in range(members):
        m = first_member + mi
        rng = np.random.Generator(np.random.PCG64([seed, m]))
        k = int(rng.integers(1, 4))
        amps = rng.uniform(0.05, 0.3, size=3)
        pos = rng.uniform(0.0, L, size=3)
        lam[mi] = 10.0 ** rng.uniform(2.0, 4.0)
        H[mi], Q[mi], KK[mi], WW[mi] = multi_soliton_state(x, amps[:k], pos[:k], L=L)
    return Workload("cfg3_ensemble", n, members, 0.0, L, ("periodic", "periodic"),
                    lam, H, Q, KK, WW, cfl=2.0, mcfl=0.5,
                    steps=200, filter_sigma=filter_sigma,
                    meta=dict(seed=seed, first_member=first_member))


def flat_rest(n: int, dx: float, h0: float = 1.0, lam: float = 500.0, noise: float = 0.0,
              seed: int = 0, members: int = 1) -> Workload:
    """Periodic rest state (h0, 0, h0^2, 0) plus optional seeded noise."""
    rng = np.random.Generator(np.random.PCG64(seed))
    sh = (members, n)
    h = h0 + noise * rng.standard_normal(sh)
    q = noise * rng.standard_normal(sh)
    K = h0 * h0 + noise * rng.standard_normal(sh)
    W = noise * rng.standard_normal(sh)
    return Workload("flat_rest", n, members, 0.0, n * dx, ("periodic", "periodic"),
                    np.full(members, lam), h, q, K, W)


def random_smooth(n: int, members: int, seed: int, dx: float = 0.1, amp: float = 0.05,
                  modes: int = 8, bc=("periodic", "periodic"), lam_range=(1e2, 1e4),
                  bathy: float = 0.0) -> Workload:
    """Seeded smooth random states (parity cases): zeta = 1 + amp * sum of periodic
    modes, u = small smooth field, eta = h (1 + small), w small; optional
    sinusoidal bathymetry of amplitude `bathy`."""
    rng = np.random.Generator(np.random.PCG64(seed))
    L = n * dx
    x = cell_centres(0.0, L, n)
    H = np.empty((members, n)); Q = np.empty((members, n))
    KK = np.empty((members, n)); WW = np.empty((members, n))
    b = None
    if bathy > 0:
        b = bathy * np.sin(2 * np.pi * 3 * x / L)
    for m in range(members):
        k = rng.integers(1, max(2, n // 128), size=modes)   # >= 128 cells per wavelength
        ph = rng.uniform(0, 2 * np.pi, size=(4, modes))
        a = rng.standard_normal((4, modes)) / np.sqrt(modes)
        if bc[0] == "periodic":
            f = [np.sum(a[j, :, None] * np.cos(2 * np.pi * k[:, None] * x[None] / L + ph[j, :, None]), 0)
                 for j in range(4)]
        else:
            # mirror-compatible fields at the ends: even (cos) for h, eta, w and odd
            # (sin) for u, so reflection ghosts continue the fields smoothly
            f = [np.sum(a[j, :, None] * (np.sin if j == 1 else np.cos)(np.pi * k[:, None] * x[None] / L), 0)
                 for j in range(4)]
        zeta = 1.0 + amp * f[0]
        h = zeta - (b if b is not None else 0.0)
        u = 0.3 * amp * f[1]
        eta = h * (1.0 + 0.01 * amp * f[2])
        w = 0.1 * amp * f[3]
        H[m] = h
        Q[m] = h * u
        KK[m] = h * eta + (1.5 * h * b if b is not None else 0.0)
        WW[m] = h * w
    lam = 10.0 ** rng.uniform(np.log10(lam_range[0]), np.log10(lam_range[1]), size=members)
    return Workload("random_smooth", n, members, 0.0, L, tuple(bc), lam, H, Q, KK, WW, b=b)


def gaussian_bell(n: int = 5000, lam: float = 100.0) -> Workload:
    """Paper's Gaussian bell: h = 1 + exp(-x^2/20) on [-200, 200], u = 0,
    eta = h, w = 0; CFL_IMEX = 2.  Boundary: transmissive."""
    x = cell_centres(-200.0, 200.0, n)
    h = 1.0 + np.exp(-x * x / 20.0)
    z = np.zeros_like(h)
    return Workload("gaussian_bell", n, 1, -200.0, 200.0, ("transmissive", "transmissive"),
                    np.array([lam]), h[None], z[None].copy(), (h * h)[None], z[None].copy(),
                    cfl=2.0, mcfl=0.5, t_end=35.0)


def lake_at_rest(n: int, lam: float, L: float = 40.0, amp: float = 0.1, h_ref: float = 0.5,
                 bc=("periodic", "periodic")) -> Workload:
    """zeta = const, u = 0, eta = h, w = 0 over smooth periodic bathymetry."""
    x = cell_centres(0.0, L, n)
    b = amp * np.sin(2 * np.pi * x / L) + 0.5 * amp * np.cos(4 * np.pi * x / L)
    h = h_ref - b
    z = np.zeros_like(h)
    K = h * (h + 1.5 * b)
    return Workload("lake_at_rest", n, 1, 0.0, L, tuple(bc), np.array([lam]), h[None],
                    z[None].copy(), K[None], z[None].copy(), b=b)


def cfg5(n: int = 1 << 28, seed: int = 7539005, lam: float = 1e4, device: str | None = None,
         first: int = 0, count: int | None = None):
    """Single large periodic domain: dx = 1/16, L = n/16; zeta = 1 + 0.05 G(x),
    G = unit-RMS sum of 64 cosine modes with distinct wavenumbers m_j uniform in
    [L/128, L/16] (wavelengths 16-128 m), A_j ~ N(0,1), phi_j ~ U[0, 2 pi);
    b = 0.2 sin(2 pi x / 128); h = zeta - b, u = 0, eta = h, w = 0,
    K = h (h + 1.5 b), W = 0; lambda = 1e4, 100 steps, CFL_IMEX 2, MCFL 0.5, A19
    filter on (the literal scheme amplifies a 1e-14 perturbation to 1e-7 in the
    100 steps at n = 2^18; filtered: 1e-10).

    Returns the cells [first, first + count) (a slab), as numpy arrays, or as
    torch tensors on `device` (fp64; used for n = 2^28, where numpy is slow)."""
    L = n / 16.0
    rng = np.random.Generator(np.random.PCG64(seed))
    lo, hi = max(1, int(L / 128)), max(2, int(L / 16))
    m = rng.choice(np.arange(lo, hi + 1), size=64, replace=False).astype(np.float64)
    A = rng.standard_normal(64)
    ph = rng.uniform(0.0, 2 * np.pi, size=64)
    A = A / np.sqrt(0.5 * np.sum(A * A))             # unit RMS of sum A_j cos(...)
    count = n - first if count is None else count
    mb = L / 128.0
    if device is None:
        x = cell_centres(0.0, L, n)[first:first + count]
        G = np.zeros(count)
        for j in range(64):
            G += A[j] * np.cos(2 * np.pi * m[j] * x / L + ph[j])
        b = 0.2 * np.sin(2 * np.pi * mb * x / L)
        zeta = 1.0 + 0.05 * G
        h = zeta - b
        z = np.zeros(count)
        out = (h, z, h * (h + 1.5 * b), z.copy(), b)
    else:
        import torch
        x = (torch.arange(first, first + count, dtype=torch.float64, device=device) + 0.5) * (L / n)
        G = torch.zeros(count, dtype=torch.float64, device=device)
        for j in range(64):
            G += A[j] * torch.cos(2 * np.pi * m[j] * x / L + ph[j])
        b = 0.2 * torch.sin(2 * np.pi * mb * x / L)
        h = 1.0 + 0.05 * G - b
        z = torch.zeros_like(h)
        out = (h, z, h * (h + 1.5 * b), z.clone(), b)
    return out, dict(n=n, L=L, lam=lam, cfl=2.0, mcfl=0.5, steps=100, seed=seed)


def cfg5_workload(n: int = 1 << 22, seed: int = 7539005, lam: float = 1e4) -> Workload:
    """cfg5 at a reduced size as a numpy Workload (parity cases)."""
    (h, q, K, W, b), meta = cfg5(n, seed, lam)
    return Workload(f"cfg5_n{n}", n, 1, 0.0, meta["L"], ("periodic", "periodic"),
                    np.array([lam]), h[None], q[None], K[None], W[None], b=b, cfl=2.0, mcfl=0.5,
                    steps=100, filter_sigma=0.25, meta=meta)


def bar_bathymetry(x, h_off: float = 0.4):
    """Submerged trapezoidal bar of cfg4 (BASELINE configs[3]): still-water depth
    0.4 offshore, slope 1:20 from x = 6 up to a 0.1-deep crest at x = 12, crest to
    x = 14, slope 1:10 down to 0.4 at x = 17, flat beyond; b = 0.4 - depth."""
    depth = np.full_like(x, h_off)
    up = (x >= 6.0) & (x < 12.0)
    depth[up] = h_off - (x[up] - 6.0) / 20.0
    depth[(x >= 12.0) & (x < 14.0)] = 0.1
    dn = (x >= 14.0) & (x < 17.0)
    depth[dn] = 0.1 + (x[dn] - 14.0) / 10.0
    return h_off - depth


def airy_wavenumber(omega: float, h0: float, g: float = G_DEFAULT) -> float:
    """Linear wave: omega^2 = g k tanh(k h0) (fixed-point iteration)."""
    k = omega * omega / g
    for _ in range(200):
        k = omega * omega / (g * math.tanh(k * h0))
    return k


def cfg4(n: int = 1 << 20, lams=(1e2, 1e3, 1e4, 1e5), L: float = 40.0) -> Workload:
    """Waves over a submerged bar: [0, 40] m, N = 2^20, bar of bar_bathymetry, lake at
    rest initially; wavemaker relaxation zone [0, 4] m (amplitude 0.01, period
    2.02 s, Airy k and phase speed) at a transmissive end x = 0 (a wall there
    conflicts with the forced velocity and grows a grid-scale mode); sponge
    [30, 40] m before a transmissive end (A10); the lambda sweep runs as 4 ensemble
    members sharing the bathymetry; CFL_IMEX 2, MCFL 0.5, 200 steps, A19 filter on.
    The bar's slope kinks make the lake at rest drift (O(dx^2) residual, A9): the
    recipe is meant for fine grids (2^16 cells and up; 2^12 blows up in ~100 steps)."""
    x = cell_centres(0.0, L, n)
    b = bar_bathymetry(x)
    h = 0.4 - b
    M = len(lams)
    H = np.tile(h, (M, 1))
    z = np.zeros_like(H)
    omega = 2 * math.pi / 2.02
    k = airy_wavenumber(omega, 0.4)
    relax = dict(x_min=0.0, level=0.4, gen_x1=4.0, gen_rate=0.1, amp=0.01, omega=omega, k=k,
                 cp=omega / k, sp_x0=30.0, sp_rate=0.1)
    return Workload("cfg4_bar", n, M, 0.0, L, ("transmissive", "transmissive"), np.array(lams, dtype=float),
                    H, z, H * (H + 1.5 * b[None]), z.copy(), b=b, cfl=2.0, mcfl=0.5, steps=200,
                    filter_sigma=0.25, meta=dict(relax=relax))
