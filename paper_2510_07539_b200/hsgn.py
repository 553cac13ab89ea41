"""Thin Python binding of libhsgn.so (include/hsgn.h): argument marshalling only.

Every step of the SI-IMEX path runs in the CUDA kernels of csrc/; this module
only passes pointers and sizes.  torch provides device memory (the workspace)
and the stream.  There is no CPU fallback: if the library is missing or no
CUDA device is present, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HSGN_LIB") or os.path.join(_PKG, "lib", "libhsgn.so")

BC = {"periodic": 0, "wall": 1, "transmissive": 2, "halo": 3}
STATUS = {0: "OK", -1: "E_INVALID", -2: "E_DRY", -3: "E_COERCIVITY", -4: "E_SINGULAR",
          -5: "E_NONFINITE", -6: "E_CUDA", -7: "E_OVERLAP", -8: "E_NOWORKSPACE", -9: "E_COMM"}


# statuses of a latched device error (a failed step: the state stays the last committed one)
DEVICE_ERRORS = (-2, -3, -5, -7)


class HsgnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"hsgn {STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Desc(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_members", C.c_int32), ("order", C.c_int32),
                ("x_min", C.c_double), ("x_max", C.c_double), ("bc_left", C.c_int32),
                ("bc_right", C.c_int32), ("tile_cells", C.c_int32), ("overlap", C.c_int32)]


class Tableau(C.Structure):
    _fields_ = [("stages", C.c_int32), ("pad_", C.c_int32), ("a_exp", (C.c_double * 2) * 2),
                ("a_imp", (C.c_double * 2) * 2), ("b", C.c_double * 2)]


class Relax(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("level", "gen_x1", "gen_rate", "amp", "omega", "k", "cp",
                                          "sp_x0", "sp_rate")]


class Diag(C.Structure):
    _fields_ = [("mass", C.c_double), ("min_h", C.c_double), ("max_abs_u", C.c_double),
                ("nu_max", C.c_double), ("t_min", C.c_double), ("t_max", C.c_double),
                ("dt_last_min", C.c_double), ("dt_last_max", C.c_double), ("rho_max", C.c_double),
                ("min_kappa", C.c_double), ("cfl_imex", C.c_double), ("mcfl", C.c_double),
                ("steps", C.c_int64), ("error_bits", C.c_int32), ("pad_", C.c_int32)]


# exported symbols (checked by tests/test_abi.py against include/hsgn.h)
SYMBOLS = ["hsgn_create", "hsgn_destroy", "hsgn_workspace_bytes", "hsgn_set_workspace",
           "hsgn_set_params", "hsgn_set_tableau", "hsgn_set_bathymetry", "hsgn_set_filter",
           "hsgn_set_relaxation",
           "hsgn_set_state", "hsgn_get_state", "hsgn_run_host", "hsgn_step", "hsgn_run_steps", "hsgn_advance_to",
           "hsgn_sync", "hsgn_run_steps_timed", "hsgn_get_diagnostics", "hsgn_launch_count", "hsgn_get_geometry",
           "hsgn_set_scheme",
           "hsgn_set_picard", "hsgn_set_well_balanced", "hsgn_set_cluster", "hsgn_get_cluster",
           "hsgn_status_string", "hsgn_last_error", "hsgn_group_create", "hsgn_group_run_steps",
           "hsgn_group_destroy", "hsgn_nccl_unique_id", "hsgn_attach_nccl",
           "hsgn_slab_xfer_count", "hsgn_slab_get", "hsgn_slab_put", "hsgn_slab_phase",
           "hsgn_run_resident", "hsgn_debug_copy"]

XFER = {"maxima": 0, "un": 1, "u1": 2, "b": 3}
PHASE = {"dt": 0, "stage1": 1, "stage2": 2, "commit": 3}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libhsgn.so and declare its signatures (no CUDA calls)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} missing: run `python -m paper_2510_07539_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, dp = C.c_void_p, C.POINTER(C.c_double)
    st = C.c_int
    sig = {
        "hsgn_create": (st, [C.POINTER(Desc), vp, C.POINTER(vp)]),
        "hsgn_destroy": (None, [vp]),
        "hsgn_workspace_bytes": (C.c_size_t, [vp]),
        "hsgn_set_workspace": (st, [vp, vp, C.c_size_t]),
        "hsgn_set_params": (st, [vp, C.c_double, dp, C.c_double, C.c_double, C.c_double]),
        "hsgn_set_tableau": (st, [vp, C.POINTER(Tableau)]),
        "hsgn_set_bathymetry": (st, [vp, vp]),
        "hsgn_set_filter": (st, [vp, C.c_double, C.c_uint32]),
        "hsgn_set_relaxation": (st, [vp, C.POINTER(Relax)]),
        "hsgn_set_state": (st, [vp, vp, vp, vp, vp, C.c_double]),
        "hsgn_get_state": (st, [vp, vp, vp, vp, vp, vp]),
        "hsgn_run_host": (st, [vp, vp, vp, vp, vp, C.c_double, C.c_int64, vp, vp, vp, vp, vp, C.c_int32]),
        "hsgn_step": (st, [vp, C.c_double, dp]),
        "hsgn_run_steps": (st, [vp, C.c_int64]),
        "hsgn_advance_to": (st, [vp, C.c_double, C.c_int64, C.POINTER(C.c_int64)]),
        "hsgn_sync": (st, [vp]),
        "hsgn_run_steps_timed": (st, [vp, C.c_int64, dp]),
        "hsgn_get_diagnostics": (st, [vp, C.POINTER(Diag)]),
        "hsgn_launch_count": (C.c_int64, [vp]),
        "hsgn_get_geometry": (st, [vp] + [C.POINTER(C.c_int32)] * 5),
        "hsgn_set_scheme": (st, [vp, C.c_int32, C.c_int32]),
        "hsgn_set_picard": (st, [vp, C.c_int32]),
        "hsgn_set_well_balanced": (st, [vp, C.c_int32]),
        "hsgn_set_cluster": (st, [vp, C.c_int32]),
        "hsgn_get_cluster": (C.c_int32, [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "hsgn_status_string": (C.c_char_p, [st]),
        "hsgn_group_create": (st, [C.POINTER(vp), C.c_int32, C.POINTER(vp)]),
        "hsgn_group_run_steps": (st, [vp, C.c_int64]),
        "hsgn_group_destroy": (None, [vp]),
        "hsgn_nccl_unique_id": (st, [C.c_char_p]),
        "hsgn_attach_nccl": (st, [vp, C.c_char_p, C.c_int32, C.c_int32]),
        "hsgn_last_error": (C.c_char_p, [vp]),
        "hsgn_slab_xfer_count": (C.c_int64, [vp, C.c_int32]),
        "hsgn_slab_get": (st, [vp, C.c_int32, vp]),
        "hsgn_slab_put": (st, [vp, C.c_int32, vp]),
        "hsgn_slab_phase": (st, [vp, C.c_int32]),
        "hsgn_run_resident": (st, [vp, C.c_int64, C.c_double, dp]),
        "hsgn_debug_copy": (st, [vp, C.c_int32, dp, C.c_int64]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def paper_tableau() -> Tableau:
    """gamma = 1 - 1/sqrt 2, c = 1/(2 gamma)."""
    g = 1.0 - 1.0 / np.sqrt(2.0)
    c = 1.0 / (2.0 * g)
    return make_tableau(2, [[0, 0], [c, 0]], [[g, 0], [1 - g, g]], [1 - g, g])


def euler_tableau() -> Tableau:
    """First-order SI step: one implicit stage with tau = dt."""
    return make_tableau(1, [[0, 0], [0, 0]], [[1.0, 0], [0, 0]], [1.0, 0])


def make_tableau(stages, aE, aI, b) -> Tableau:
    T = Tableau()
    T.stages = stages
    for i in range(2):
        for j in range(2):
            T.a_exp[i][j] = float(aE[i][j])
            T.a_imp[i][j] = float(aI[i][j])
        T.b[i] = float(b[i])
    return T


def _ptr(a):
    """Raw pointer of a torch tensor (device or host) or a numpy array."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.dtype == np.float64 and a.flags.c_contiguous
        return a.ctypes.data
    import torch
    assert a.dtype == torch.float64 and a.is_contiguous()
    return a.data_ptr()


@dataclass
class Geometry:
    tile_cells: int
    overlap: int
    tiles_per_member: int
    threads: int
    max_rows: int


class Solver:
    """One context: `members` independent 1-D domains of `n` cells each."""

    def __init__(self, n: int, members: int = 1, x_min: float = 0.0, x_max: float = 1.0,
                 bc=("periodic", "periodic"), order: int = 2, tile_cells: int = 0,
                 overlap: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the hSGN path has no CPU fallback")
        self.L = load_library()
        self.n, self.members = int(n), int(members)
        self.dx = (x_max - x_min) / n
        self._torch = torch
        # a dedicated non-default stream: CUDA graphs cannot capture the legacy stream
        self.stream = stream if stream is not None else torch.cuda.Stream()
        d = Desc(n_cells=n, n_members=members, order=order, x_min=x_min, x_max=x_max,
                 bc_left=BC[bc[0]], bc_right=BC[bc[1]], tile_cells=tile_cells, overlap=overlap)
        h = C.c_void_p()
        self._chk(self.L.hsgn_create(C.byref(d), C.c_void_p(self.stream.cuda_stream), C.byref(h)),
                  ctx=False)
        self.ctx = h
        nbytes = self.L.hsgn_workspace_bytes(self.ctx)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        # the library works on self.stream: order it after torch's stream (the
        # memory may just have been released there) and tell the allocator
        self.workspace.record_stream(self.stream)
        self.stream.wait_stream(torch.cuda.current_stream())
        self._chk(self.L.hsgn_set_workspace(self.ctx, C.c_void_p(self.workspace.data_ptr()), nbytes))
        self._keep = []

    # -- plumbing ----------------------------------------------------------
    def _chk(self, st, ctx=True):
        if st != 0:
            msg = self.L.hsgn_last_error(self.ctx).decode() if ctx else ""
            raise HsgnError(st, msg or self.L.hsgn_status_string(st).decode())

    def close(self):
        if getattr(self, "ctx", None):
            self.L.hsgn_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def geometry(self) -> Geometry:
        v = [C.c_int32() for _ in range(5)]
        self._chk(self.L.hsgn_get_geometry(self.ctx, *[C.byref(x) for x in v]))
        return Geometry(*[x.value for x in v])

    def set_scheme(self, scheme: str = "si", stages: int = 2) -> None:
        """"si" (IMEX), "explicit" (hSGN) or "sgn" (classical
        SGN); stages 1 Euler, 2 Heun for the last two."""
        code = {"si": 0, "explicit": 1, "sgn": 2}[scheme]
        self._chk(self.L.hsgn_set_scheme(self.ctx, code, stages))

    def set_picard(self, passes: int) -> None:
        """A24 Picard passes of the SI depth solve (0 = the paper's linearised stage)."""
        self._chk(self.L.hsgn_set_picard(self.ctx, int(passes)))

    def set_well_balanced(self, on: bool = True) -> None:
        """A25 exactly well-balanced face form of the SI stage (default off: the paper's)."""
        self._chk(self.L.hsgn_set_well_balanced(self.ctx, 1 if on else 0))

    def set_cluster(self, mode) -> None:
        """Exact depth solve across tiles (hsgn_set_cluster): 1/True = cluster
        kernels whenever the member fits, 3 = tile-level SPIKE, 0/False = never
        (overlapped tiles), 2 = auto (default: exact paths only for
        material-CFL-only stepping)."""
        self._chk(self.L.hsgn_set_cluster(self.ctx, int(mode)))

    @property
    def cluster(self):
        """(C, tile rows) if the next step runs on the cluster kernels, else None."""
        a, b = C.c_int32(), C.c_int32()
        on = int(self.L.hsgn_get_cluster(self.ctx, C.byref(a), C.byref(b)))
        return (a.value, b.value) if on == 1 else None

    @property
    def spike(self):
        """(tiles, tile rows) if the next step runs on tile-level SPIKE, else None."""
        a, b = C.c_int32(), C.c_int32()
        on = int(self.L.hsgn_get_cluster(self.ctx, C.byref(a), C.byref(b)))
        return (a.value, b.value) if on == 2 else None

    @property
    def launches(self) -> int:
        return int(self.L.hsgn_launch_count(self.ctx))

    # -- parameters ----------------------------------------------------------
    def set_params(self, g=9.81, lam=500.0, cfl=2.0, mcfl=0.5, h_min=1e-8):
        lam = np.ascontiguousarray(np.broadcast_to(np.asarray(lam, dtype=np.float64),
                                                   (self.members,)))
        self._chk(self.L.hsgn_set_params(self.ctx, g, lam.ctypes.data_as(C.POINTER(C.c_double)),
                                         cfl, mcfl, h_min))

    def set_tableau(self, tab: Tableau):
        self._chk(self.L.hsgn_set_tableau(self.ctx, C.byref(tab)))

    def set_bathymetry(self, b):
        if b is not None:
            b = self._as_f64(b)
            self._keep.append(b)
            # a device tensor may still be being written on torch's stream: the
            # library copies on the solver's stream
            self.stream.wait_stream(self._torch.cuda.current_stream())
        self._chk(self.L.hsgn_set_bathymetry(self.ctx, C.c_void_p(_ptr(b)) if b is not None else None))

    def set_relaxation(self, relax: dict | None):
        """A10 wavemaker / sponge zones: keys level, gen_x1, gen_rate, amp, omega, k,
        cp, sp_x0, sp_rate (see include/hsgn.h); None disables them."""
        if relax is None:
            self._chk(self.L.hsgn_set_relaxation(self.ctx, None))
        else:
            r = Relax(**{k: float(v) for k, v in relax.items()})
            self._chk(self.L.hsgn_set_relaxation(self.ctx, C.byref(r)))

    def set_filter(self, sigma: float, mask: int = 0b1010):
        self._chk(self.L.hsgn_set_filter(self.ctx, float(sigma), mask if sigma > 0 else 0))

    # -- state ------------------------------------------------------------
    def _as_f64(self, a):
        if isinstance(a, np.ndarray):
            return np.ascontiguousarray(a, dtype=np.float64)
        return a.contiguous().to(self._torch.float64)

    def set_state(self, h, q, K, W, t0: float = 0.0):
        arrs = [self._as_f64(a) for a in (h, q, K, W)]
        for a in arrs:
            assert a.size == self.n * self.members if isinstance(a, np.ndarray) else a.numel() == self.n * self.members
        self.stream.wait_stream(self._torch.cuda.current_stream())
        self._chk(self.L.hsgn_set_state(self.ctx, *[C.c_void_p(_ptr(a)) for a in arrs], t0))

    def get_state(self, device: bool = True, check: bool = True):
        """Return (h, q, K, W) as [members, n] tensors (device) or numpy arrays, and t[members].
        A latched device error (a failed step) raises unless check=False; the copy is
        made either way and holds the last committed state (include/hsgn.h)."""
        torch = self._torch
        if device:
            out = [torch.empty((self.members, self.n), dtype=torch.float64, device="cuda") for _ in range(4)]
            self.stream.wait_stream(torch.cuda.current_stream())
        else:
            out = [np.empty((self.members, self.n)) for _ in range(4)]
        t = np.empty(self.members)
        st = self.L.hsgn_get_state(self.ctx, *[C.c_void_p(_ptr(a)) for a in out], C.c_void_p(t.ctypes.data))
        if st != 0 and (check or st not in DEVICE_ERRORS):
            self._chk(st)
        return out, t

    def run_host(self, h, q, K, W, n_steps: int, out=None, chunks: int = 8, t0: float = 0.0):
        """hsgn_run_host: a whole job from host arrays (numpy or CPU tensors, pinned
        for copy/compute overlap) -- n_steps steps of every member, pipelined over
        member chunks.  Returns ((h, q, K, W) written into `out` or new numpy
        arrays of shape [members, n], t[members])."""
        N = self.n * self.members
        arrs = [self._as_f64(a) for a in (h, q, K, W)]
        for a in arrs:
            assert (a.size if isinstance(a, np.ndarray) else a.numel()) == N
        if out is None:
            out = [np.empty((self.members, self.n)) for _ in range(4)]
        t = np.empty(self.members)
        self.stream.wait_stream(self._torch.cuda.current_stream())
        self._chk(self.L.hsgn_run_host(self.ctx, *[C.c_void_p(_ptr(a)) for a in arrs], float(t0),
                                       int(n_steps), *[C.c_void_p(_ptr(o)) for o in out],
                                       C.c_void_p(t.ctypes.data), int(chunks)))
        return out, t

    # -- stepping ------------------------------------------------------------
    def step(self, dt: float = 0.0, return_dt: bool = False):
        if return_dt:
            d = np.empty(self.members)
            self._chk(self.L.hsgn_step(self.ctx, dt, d.ctypes.data_as(C.POINTER(C.c_double))))
            return d
        self._chk(self.L.hsgn_step(self.ctx, dt, None))

    def debug_copy(self, which: int, count: int) -> np.ndarray:
        """hsgn_debug_copy: an internal SPIKE array (development aid)"""
        out = np.empty(count)
        self._chk(self.L.hsgn_debug_copy(self.ctx, int(which), out.ctypes.data_as(C.POINTER(C.c_double)), count))
        return out

    def run_resident(self, n_steps: int, t_end: float = 0.0) -> float:
        """hsgn_run_resident: n_steps steps with every member resident in its
        cluster's shared memory (one launch), the last step clipped to t_end if
        t_end > 0; returns the device ms."""
        ms = C.c_double()
        self._chk(self.L.hsgn_run_resident(self.ctx, int(n_steps), float(t_end), C.byref(ms)))
        return ms.value

    def run_steps(self, n_steps: int):
        self._chk(self.L.hsgn_run_steps(self.ctx, int(n_steps)))

    def run_steps_timed(self, n_steps: int, total: bool = False):
        """n steps as one CUDA graph with event nodes between the kernels; returns
        the summed device ms per stage kind (stage 1, stage 2) and, with
        total=True, also the device ms of the whole n steps."""
        ms = np.zeros(3)
        self._chk(self.L.hsgn_run_steps_timed(self.ctx, int(n_steps),
                                              ms.ctypes.data_as(C.POINTER(C.c_double))))
        return (float(ms[0]), float(ms[1]), float(ms[2])) if total else (float(ms[0]), float(ms[1]))

    def advance_to(self, t_end: float, max_steps: int = 1 << 40) -> int:
        s = C.c_int64()
        self._chk(self.L.hsgn_advance_to(self.ctx, t_end, max_steps, C.byref(s)))
        return s.value

    def sync(self):
        self._chk(self.L.hsgn_sync(self.ctx))

    def attach_nccl(self, unique_id: bytes, rank: int, world: int):
        """Slab of a domain sharded over `world` processes (one GPU each)."""
        assert len(unique_id) == 128
        self._chk(self.L.hsgn_attach_nccl(self.ctx, unique_id, rank, world))

    # -- host-staged slab transport (include/hsgn.h) -------------------------
    def slab_get(self, what: str) -> np.ndarray:
        """Boundary data this slab sends ("un", "u1", "b": [left | right]) or its
        dt maxima ("maxima", uint64 bit patterns)."""
        n = int(self.L.hsgn_slab_xfer_count(self.ctx, XFER[what]))
        if n < 0:
            raise HsgnError(-1, "slab_get: not a slab context")
        out = np.empty(n, dtype=np.uint64 if what == "maxima" else np.float64)
        self._chk(self.L.hsgn_slab_get(self.ctx, XFER[what], C.c_void_p(out.ctypes.data)))
        return out

    def slab_put(self, what: str, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, dtype=np.uint64 if what == "maxima" else np.float64)
        assert data.size == int(self.L.hsgn_slab_xfer_count(self.ctx, XFER[what]))
        self._chk(self.L.hsgn_slab_put(self.ctx, XFER[what], C.c_void_p(data.ctypes.data)))

    def slab_phase(self, phase: str) -> None:
        self._chk(self.L.hsgn_slab_phase(self.ctx, PHASE[phase]))

    def diagnostics(self) -> dict:
        d = Diag()
        self._chk(self.L.hsgn_get_diagnostics(self.ctx, C.byref(d)))
        return {k: getattr(d, k) for k, _ in Diag._fields_ if k != "pad_"}


def solver_for(w, **kw) -> Solver:
    """Build a Solver for a workloads.Workload (state, params, bathymetry, filter)."""
    s = Solver(w.n, w.members, w.x_min, w.x_max, bc=w.bc, **kw)
    s.set_params(w.g, w.lam, w.cfl, w.mcfl)
    if w.b is not None:
        s.set_bathymetry(w.b)
    if w.filter_sigma > 0:
        s.set_filter(w.filter_sigma)
    if w.meta.get("relax"):
        s.set_relaxation({k: v for k, v in w.meta["relax"].items() if k != "x_min"})
    s.set_state(w.h.reshape(-1), w.q.reshape(-1), w.K.reshape(-1), w.W.reshape(-1))
    return s


def nccl_unique_id() -> bytes:
    L = load_library()
    buf = C.create_string_buffer(128)
    st = L.hsgn_nccl_unique_id(buf)
    if st != 0:
        raise HsgnError(st, "ncclGetUniqueId")
    return buf.raw


class Group:
    """In-process slab group: Solvers (ring order) sharing one stream, stepped in
    lockstep with device-to-device halo exchange (C ABI hsgn_group_*)."""

    def __init__(self, solvers):
        self.solvers = list(solvers)
        self.L = load_library()
        arr = (C.c_void_p * len(self.solvers))(*[sv.ctx.value for sv in self.solvers])
        h = C.c_void_p()
        st = self.L.hsgn_group_create(arr, len(self.solvers), C.byref(h))
        if st != 0:
            raise HsgnError(st, self.L.hsgn_last_error(self.solvers[0].ctx).decode())
        self.g = h

    def run_steps(self, n_steps: int):
        st = self.L.hsgn_group_run_steps(self.g, int(n_steps))
        if st != 0:
            raise HsgnError(st, self.L.hsgn_last_error(self.solvers[0].ctx).decode())

    def close(self):
        if getattr(self, "g", None):
            self.L.hsgn_group_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_solvers(w, parts, stream=None, align=1, **kw):
    """Split a 1-member Workload into `parts` contiguous slabs (sizes differ by at
    most `align` cells, edges multiples of `align`; SPIKE across slabs needs
    multiples of 4) sharing one stream; returns (solvers, bounds)."""
    import torch
    assert w.members == 1
    stream = stream if stream is not None else torch.cuda.Stream()
    edges = [align * round(i * w.n / (parts * align)) for i in range(parts)] + [w.n]
    out = []
    for i in range(parts):
        a, b = edges[i], edges[i + 1]
        left = "halo" if (i > 0 or w.bc[0] == "periodic") else w.bc[0]
        right = "halo" if (i < parts - 1 or w.bc[1] == "periodic") else w.bc[1]
        sv = Solver(b - a, 1, w.x_min + a * w.dx, w.x_min + b * w.dx, bc=(left, right),
                    stream=stream, **kw)
        sv.set_params(w.g, w.lam, w.cfl, w.mcfl)
        if w.b is not None:
            sv.set_bathymetry(np.ascontiguousarray(w.b[a:b]))
        if w.filter_sigma > 0:
            sv.set_filter(w.filter_sigma)
        sv.set_state(*[np.ascontiguousarray(f[0, a:b]) for f in (w.h, w.q, w.K, w.W)])
        out.append(sv)
    return out, edges
