"""ctypes wrapper of the CPU fp64 oracle (oracle/hsgn_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py.  The product package
(paper_2510_07539_b200) never imports this module.

The wrapper only marshals numpy arrays; every arithmetic step of the method
lives in hsgn_oracle.c (each function there cites the PAPER.md passage it
follows).  Parity status of each function: see the header of hsgn_oracle.c
and DESIGN.md section 4.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hsgn_oracle.c")
_LIB = os.path.join(_HERE, "build", "libhsgn_oracle.so")
_LIB_FMA = os.path.join(_HERE, "build", "libhsgn_oracle_fma.so")
_lock = threading.Lock()
_lib = None
_libs = {}

BC_PERIODIC, BC_WALL, BC_TRANSMISSIVE = 0, 1, 2
OK, E_INVALID, E_DRY, E_COERCIVITY, E_SINGULAR, E_NONFINITE = 0, -1, -2, -3, -4, -5

GAMMA = 1.0 - 1.0 / np.sqrt(2.0)


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"oracle status {status} {what}")
        self.status = status


class Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("bc_left", C.c_int32), ("bc_right", C.c_int32),
        ("order", C.c_int32), ("dx", C.c_double), ("g", C.c_double),
        ("lam", C.c_double), ("h_min", C.c_double), ("b", C.POINTER(C.c_double)),
        ("filter_sigma", C.c_double), ("filter_mask", C.c_int32), ("pad_", C.c_int32),
        ("x_min", C.c_double), ("level", C.c_double), ("gen_x1", C.c_double),
        ("gen_rate", C.c_double), ("amp", C.c_double), ("omega", C.c_double), ("k", C.c_double),
        ("cp", C.c_double), ("sp_x0", C.c_double), ("sp_rate", C.c_double),
        ("picard", C.c_int32), ("wb", C.c_int32),
    ]


class Tableau(C.Structure):
    _fields_ = [("stages", C.c_int32), ("pad_", C.c_int32),
                ("aE", (C.c_double * 2) * 2), ("aI", (C.c_double * 2) * 2),
                ("b", C.c_double * 2)]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc, no FMA contraction, no fast-math.
    HSGN_ORACLE_LIB overrides the library path (used by tools/mutation_check.py)."""
    if os.environ.get("HSGN_ORACLE_LIB"):
        return os.environ["HSGN_ORACLE_LIB"]
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def build_fma(force: bool = False) -> str:
    """The SAME source compiled with FMA contraction (-ffp-contract=fast
    -march=native): a second fp64 rounding of the identical algorithm.  Used
    only to measure the rounding floor of the parity metric (reading A17):
    oracle vs oracle-fma differences are what any two correct fp64
    implementations may differ by."""
    os.makedirs(os.path.dirname(_LIB_FMA), exist_ok=True)
    if force or not os.path.exists(_LIB_FMA) or os.path.getmtime(_LIB_FMA) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-ffp-contract=fast", "-march=native",
                               "-fno-fast-math", "-fPIC", "-shared", "-o", _LIB_FMA, _SRC, "-lm"])
    return _LIB_FMA


def lib(variant: str = "plain"):
    global _lib
    with _lock:
        if variant not in _libs:
            L = C.CDLL(build() if variant == "plain" else build_fma())
            dp = C.POINTER(C.c_double)
            P, T = C.POINTER(Problem), C.POINTER(Tableau)
            L.orc_celerity.restype = C.c_double
            L.orc_celerity.argtypes = [C.c_double] * 4
            L.orc_coeffs.restype = None
            L.orc_coeffs.argtypes = [C.c_double] * 6 + [dp]
            for f in (L.orc_thomas, L.orc_cyclic_thomas):
                f.restype = C.c_int
                f.argtypes = [C.c_int, dp, dp, dp, dp, dp]
            L.orc_stage.restype = C.c_int
            L.orc_stage.argtypes = [P] + [dp] * 8 + [C.c_double] + [dp] * 5
            L.orc_step.restype = C.c_int
            L.orc_step.argtypes = [P, T, C.c_double] + [dp] * 5
            L.orc_step_t.restype = C.c_int
            L.orc_step_t.argtypes = [P, T, C.c_double, C.c_double] + [dp] * 5
            L.orc_dt.restype = C.c_int
            L.orc_dt.argtypes = [P, C.c_double, C.c_double] + [dp] * 6
            L.orc_run.restype = C.c_int
            L.orc_run.argtypes = [P, T, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_int64] + [dp] * 5 + [C.POINTER(C.c_int64), dp]
            L.orc_tableau_weights.restype = C.c_int
            L.orc_tableau_weights.argtypes = [T, dp, dp]
            L.orc_rusanov_face.restype = None
            L.orc_rusanov_face.argtypes = [dp, dp, dp]
            L.orc_explicit_rhs.restype = C.c_int
            L.orc_explicit_rhs.argtypes = [P] + [dp] * 8
            L.orc_explicit_step_t.restype = C.c_int
            L.orc_explicit_step_t.argtypes = [P, C.c_int, C.c_double, C.c_double] + [dp] * 4
            L.orc_explicit_run.restype = C.c_int
            L.orc_explicit_run.argtypes = [P, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_int64] + [dp] * 5 + [C.POINTER(C.c_int64)]
            L.orc_sgn_rhs.restype = C.c_int
            L.orc_sgn_rhs.argtypes = [P] + [dp] * 4
            L.orc_sgn_step.restype = C.c_int
            L.orc_sgn_step.argtypes = [P, C.c_int, C.c_double, dp, dp]
            L.orc_sgn_dt.restype = C.c_int
            L.orc_sgn_dt.argtypes = [P, C.c_double, dp, dp, dp]
            L.orc_sgn_run.restype = C.c_int
            L.orc_sgn_run.argtypes = [P, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_int64, dp, dp, dp, C.POINTER(C.c_int64)]
            L.orc_mass.restype = C.c_double
            L.orc_mass.argtypes = [C.c_int, C.c_double, dp]
            _libs[variant] = L
            if variant == "plain":
                _lib = L
    return _libs[variant]


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def paper_tableau() -> Tableau:
    """Double Butcher tableau of P:371-386 (gamma = 1 - 1/sqrt2, c = 1/(2 gamma))."""
    g = GAMMA
    c = 1.0 / (2.0 * g)
    return make_tableau(2, [[0.0, 0.0], [c, 0.0]], [[g, 0.0], [1.0 - g, g]], [1.0 - g, g])


def euler_tableau() -> Tableau:
    """First-order SI: one implicit stage, tau = dt."""
    return make_tableau(1, [[0.0, 0.0], [0.0, 0.0]], [[1.0, 0.0], [0.0, 0.0]], [1.0, 0.0])


def make_tableau(stages, aE, aI, b) -> Tableau:
    T = Tableau()
    T.stages = stages
    for i in range(2):
        for j in range(2):
            T.aE[i][j] = aE[i][j]
            T.aI[i][j] = aI[i][j]
        T.b[i] = b[i]
    return T


class Oracle:
    """One 1-D domain (or one ensemble member) on the host."""

    def __init__(self, n, dx, g=9.81, lam=500.0, bc=("periodic", "periodic"), order=2,
                 h_min=1e-8, b=None, filter_sigma=0.0, filter_mask=0b1010, tableau=None,
                 relax=None, picard=0, wb=False, variant="plain"):
        """relax: dict(x_min, level, gen_x1, gen_rate, amp, omega, k, cp, sp_x0, sp_rate)
        for the A10 wavemaker / sponge zones (cfg4).  variant="fma": the same
        oracle built with FMA contraction (rounding-floor measurements, A17)."""
        self.L = lib(variant)
        codes = {"periodic": BC_PERIODIC, "wall": BC_WALL, "transmissive": BC_TRANSMISSIVE}
        self._b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        self.P = Problem(n=n, bc_left=codes[bc[0]], bc_right=codes[bc[1]], order=order,
                         dx=dx, g=g, lam=lam, h_min=h_min,
                         b=_p(self._b) if self._b is not None else None,
                         filter_sigma=filter_sigma, filter_mask=filter_mask, picard=picard,
                         wb=1 if wb else 0,
                         **(relax or {}))
        self.T = tableau if tableau is not None else paper_tableau()

    # -- pieces ---------------------------------------------------------
    def stage(self, E, R, tau):
        E = [np.ascontiguousarray(a, dtype=np.float64) for a in E]
        R = [np.ascontiguousarray(a, dtype=np.float64) for a in R]
        O = [np.empty(self.P.n) for _ in range(4)]
        mb = C.c_double()
        st = self.L.orc_stage(C.byref(self.P), *[_p(a) for a in E], *[_p(a) for a in R],
                              tau, *[_p(a) for a in O], C.byref(mb))
        if st != OK:
            raise OracleError(st, "stage")
        return O, mb.value

    def step(self, U, dt, t=0.0):
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        mb = C.c_double()
        st = self.L.orc_step_t(C.byref(self.P), C.byref(self.T), t, dt, *[_p(a) for a in U],
                               C.byref(mb))
        if st != OK:
            raise OracleError(st, "step")
        return U

    def dt(self, U, cfl, mcfl):
        h, q, K = [np.ascontiguousarray(a, dtype=np.float64) for a in U[:3]]
        d, nu, um = C.c_double(), C.c_double(), C.c_double()
        st = self.L.orc_dt(C.byref(self.P), cfl, mcfl, _p(h), _p(q), _p(K), C.byref(d),
                           C.byref(nu), C.byref(um))
        if st != OK:
            raise OracleError(st, "dt")
        return d.value, nu.value, um.value

    def run(self, U, cfl=2.0, mcfl=0.5, steps=None, t0=0.0, t_end=None, dt_fixed=0.0):
        """Advance; returns (U, t, steps, min_beta).  Exactly `steps` steps when
        t_end is None, else until t_end (last step clipped)."""
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        tout, sout, mb = C.c_double(), C.c_int64(), C.c_double()
        max_steps = steps if steps is not None else (1 << 62)
        te = t_end if t_end is not None else t0 - 1.0
        st = self.L.orc_run(C.byref(self.P), C.byref(self.T), cfl, mcfl, dt_fixed, t0, te,
                            max_steps, *[_p(a) for a in U], C.byref(tout), C.byref(sout),
                            C.byref(mb))
        if st != OK:
            raise OracleError(st, f"run (after {sout.value} steps)")
        return U, tout.value, sout.value, mb.value


    # -- explicit hSGN scheme -----------------------------------
    def explicit_rhs(self, U):
        """L(U) of the explicit scheme P:444-458 (flat bottom)."""
        U = [np.ascontiguousarray(a, dtype=np.float64) for a in U]
        O = [np.empty(self.P.n) for _ in range(4)]
        st = self.L.orc_explicit_rhs(C.byref(self.P), *[_p(a) for a in U], *[_p(a) for a in O])
        if st != OK:
            raise OracleError(st, "explicit_rhs")
        return O

    def explicit_step(self, U, dt, stages=2, t=0.0):
        """One explicit step: stages 1 = forward Euler, 2 = Heun."""
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        st = self.L.orc_explicit_step_t(C.byref(self.P), stages, t, dt, *[_p(a) for a in U])
        if st != OK:
            raise OracleError(st, "explicit_step")
        return U

    def explicit_run(self, U, cfl=0.4, stages=2, steps=None, t0=0.0, t_end=None, dt_fixed=0.0):
        """Advance with dt = CFL_EX dx / mu_max; returns (U, t, steps)."""
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        tout, sout = C.c_double(), C.c_int64()
        max_steps = steps if steps is not None else (1 << 62)
        te = t_end if t_end is not None else t0 - 1.0
        st = self.L.orc_explicit_run(C.byref(self.P), stages, cfl, dt_fixed, t0, te, max_steps,
                                     *[_p(a) for a in U], C.byref(tout), C.byref(sout))
        if st != OK:
            raise OracleError(st, f"explicit_run (after {sout.value} steps)")
        return U, tout.value, sout.value


    # -- classical SGN scheme -----------------------------------
    def sgn_rhs(self, h, q):
        h = np.ascontiguousarray(h, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        Lh, Lq = np.empty(self.P.n), np.empty(self.P.n)
        st = self.L.orc_sgn_rhs(C.byref(self.P), _p(h), _p(q), _p(Lh), _p(Lq))
        if st != OK:
            raise OracleError(st, "sgn_rhs")
        return Lh, Lq

    def sgn_step(self, U, dt, stages=2):
        """One SGN step on (h, q[, K, W]); K, W are carried unchanged."""
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        st = self.L.orc_sgn_step(C.byref(self.P), stages, dt, _p(U[0]), _p(U[1]))
        if st != OK:
            raise OracleError(st, "sgn_step")
        return U

    def sgn_dt(self, U, cfl):
        h, q = [np.ascontiguousarray(a, dtype=np.float64) for a in U[:2]]
        d = C.c_double()
        st = self.L.orc_sgn_dt(C.byref(self.P), cfl, _p(h), _p(q), C.byref(d))
        if st != OK:
            raise OracleError(st, "sgn_dt")
        return d.value

    def sgn_run(self, U, cfl=0.9, stages=2, steps=None, t0=0.0, t_end=None, dt_fixed=0.0):
        U = [np.array(a, dtype=np.float64, copy=True) for a in U]
        tout, sout = C.c_double(), C.c_int64()
        max_steps = steps if steps is not None else (1 << 62)
        te = t_end if t_end is not None else t0 - 1.0
        st = self.L.orc_sgn_run(C.byref(self.P), stages, cfl, dt_fixed, t0, te, max_steps,
                                _p(U[0]), _p(U[1]), C.byref(tout), C.byref(sout))
        if st != OK:
            raise OracleError(st, f"sgn_run (after {sout.value} steps)")
        return U, tout.value, sout.value


def coeffs(g, lam, tau, h, H, Hdag):
    out = np.empty(6)
    lib().orc_coeffs(g, lam, tau, h, H, Hdag, _p(out))
    return dict(zip(("alpha", "a2", "beta1", "beta2", "beta", "delta"), out))


def rusanov_face(vm, vp):
    vm = np.ascontiguousarray(vm, dtype=np.float64)
    vp = np.ascontiguousarray(vp, dtype=np.float64)
    out = np.empty(3)
    lib().orc_rusanov_face(_p(vm), _p(vp), _p(out))
    return out


def celerity(g, lam, h, H):
    return lib().orc_celerity(g, lam, h, H)


def thomas(lo, di, up, rhs, cyclic=False):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (lo, di, up, rhs)]
    x = np.empty(len(arrs[1]))
    f = lib().orc_cyclic_thomas if cyclic else lib().orc_thomas
    st = f(len(x), *[_p(a) for a in arrs], _p(x))
    if st != OK:
        raise OracleError(st, "thomas")
    return x


def tableau_weights(T):
    a, b = C.c_double(), C.c_double()
    st = lib().orc_tableau_weights(C.byref(T), C.byref(a), C.byref(b))
    if st != OK:
        raise OracleError(st, "tableau")
    return a.value, b.value


def mass(h, dx):
    h = np.ascontiguousarray(h, dtype=np.float64)
    return lib().orc_mass(len(h), dx, _p(h))


def run_members(members, threads=None, explicit=False, sgn=False, **kw):
    """Run independent ensemble members on host threads (ctypes releases the GIL).
    members: list of (Oracle, U).  Returns list of results of Oracle.run (or of
    Oracle.explicit_run with explicit=True)."""
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=threads) as ex:
        if sgn:
            return list(ex.map(lambda m: m[0].sgn_run(m[1], **kw), members))
        if explicit:
            return list(ex.map(lambda m: m[0].explicit_run(m[1], **kw), members))
        return list(ex.map(lambda m: m[0].run(m[1], **kw), members))
