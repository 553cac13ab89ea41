"""GPU parity of the tile-level SPIKE path (hsgn_cluster.cuh CL_MODE_TIPS /
FINISH, sep_solve_kernel, filter_fix_kernel): the depth system of P:509-512
solved exactly across the tiles of members of any size, against the oracle
(metric A17, see test_gpu_parity.py) and against the other GPU paths."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, compare, field_scales, rel_err
from tests.test_gpu_parity import gpu_solver as _gpu_solver

pytestmark = pytest.mark.gpu


def gpu_solver(w, **kw):
    """a solver on tile-level SPIKE (mode 3)"""
    s = _gpu_solver(w, **kw)
    s.set_cluster(3)
    return s


@pytest.mark.parametrize("n,bc,G", [(4096, "periodic", 8), (3000, "wall", 6), (1 << 16, "periodic", 128),
                                    (512, "periodic", 1), (1000, "transmissive", 2), (64, "periodic", 1), (16, "wall", 1),
                                    (20000, "wall", 40)])
@pytest.mark.parametrize("filt", [0.25, 0.0])
def test_spike_steps(n, bc, G, filt):
    w = W.random_smooth(n, 2, seed=n + G, amp=0.08, bc=(bc, bc))
    w.filter_sigma = filt
    s = gpu_solver(w)
    assert s.spike is not None and s.spike[0] == G, s.spike
    s.step()
    compare(w, s, range(2), steps=1, floor=True)
    s.run_steps(19)
    compare(w, s, range(2), steps=20, tol=1e-10)


@pytest.mark.parametrize("order", [1, 2])
def test_spike_bathymetry_walls_and_order(order):
    w = W.random_smooth(6000, 2, seed=41, amp=0.05, bc=("wall", "wall"), bathy=0.08)
    w.filter_sigma = 0.25
    s = gpu_solver(w, order=order)
    assert s.spike is not None
    s.step()
    compare(w, s, range(2), steps=1, order=order)
    s.run_steps(9)
    compare(w, s, range(2), steps=10, tol=1e-10, order=order)


def test_spike_first_order_tableau():
    from paper_2510_07539_b200 import hsgn as hs
    w = W.random_smooth(3000, 2, seed=8, amp=0.05)
    s = gpu_solver(w, tableau=hs.euler_tableau(), order=1)
    assert s.spike is not None
    s.run_steps(5)
    compare(w, s, range(2), steps=5, order=1, tableau=O.euler_tableau(), tol=1e-10)


def test_spike_cfg5_recipe_and_equal_to_tiles():
    """cfg5 recipe (bathymetry, filter, lam = 1e4) on 2^18 cells: SPIKE == oracle,
    and == the overlapped tiles to round-off (same arithmetic, different
    exact solves)"""
    w = W.cfg5_workload(1 << 18)
    a = gpu_solver(w)
    b = _gpu_solver(w)
    b.set_cluster(0)
    assert a.spike == (512, 512) and b.spike is None
    a.step()
    compare(w, a, [0], steps=1, floor=True)
    a.run_steps(9)
    b.run_steps(10)
    (x, tx), (y, ty) = a.get_state(device=False), b.get_state(device=False)
    ref = [f[0] for f in y]
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), b=w.b).dt(ref, w.cfl, w.mcfl)[0]
    assert rel_err([f[0] for f in x], ref, field_scales(ref, float(w.lam[0]), dt)) <= 1e-12
    assert abs(tx[0] - ty[0]) <= 1e-13 * ty[0]


@pytest.mark.parametrize("n,bc,G", [(1 << 20, "periodic", 2048), (600000, "wall", 1172)])
def test_spike_large_members_1024_thread_separator_solve(n, bc, G):
    """more than 1024 tiles per member: the separator system is solved by the
    1024-thread sep_solve_kernel (chunks of <= 2 separators per thread here)"""
    w = W.random_smooth(n, 1, seed=n, amp=0.08, bc=(bc, bc))
    w.filter_sigma = 0.25
    s = gpu_solver(w)
    assert s.spike == (G, 512), s.spike
    s.step()
    compare(w, s, [0], steps=1, floor=True)
    s.run_steps(4)
    compare(w, s, [0], steps=5, tol=1e-10)
    b = _gpu_solver(w)
    b.set_cluster(0)
    b.run_steps(5)
    (x, tx), (y, ty) = s.get_state(device=False), b.get_state(device=False)
    ref = [f[0] for f in y]
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc).dt(ref, w.cfl, w.mcfl)[0]
    assert rel_err([f[0] for f in x], ref, field_scales(ref, float(w.lam[0]), dt)) <= 1e-12
    assert abs(tx[0] - ty[0]) <= 1e-13 * ty[0]


def test_spike_equals_cluster():
    w = W.random_smooth(4096, 3, seed=12, amp=0.1)
    w.filter_sigma = 0.25
    a, b = gpu_solver(w), _gpu_solver(w)
    b.set_cluster(1)
    assert a.spike == (8, 512) and b.cluster == (8, 512)
    a.run_steps(10)
    b.run_steps(10)
    (x, tx), (y, ty) = a.get_state(device=False), b.get_state(device=False)
    for m in range(3):
        ref = [f[m] for f in y]
        dt = O.Oracle(w.n, w.dx, lam=float(w.lam[m])).dt(ref, w.cfl, w.mcfl)[0]
        assert rel_err([f[m] for f in x], ref, field_scales(ref, float(w.lam[m]), dt)) <= 1e-12


def test_spike_relaxation_zones_cfg4():
    """cfg4 recipe (bar, wavemaker + sponge zones, 4 lambdas) on 2^16 cells"""
    w = W.cfg4(n=1 << 16)
    s = gpu_solver(w)
    assert s.spike is not None
    s.step()
    compare(w, s, range(4), steps=1)
    s.run_steps(59)
    compare(w, s, range(4), steps=60, tol=1e-10)


def test_auto_mode_mcfl_only_large_domain_uses_spike_and_matches_oracle():
    """material-CFL-only stepping (cfl_imex off) on a walled 2^16-cell domain:
    auto mode takes the exact tile-level SPIKE (the member does not fit a
    cluster); a large step (MCFL 0.5 with slow flow: rho ~ 10^2) still
    matches the oracle"""
    w = W.cfg2(100.0, n=1 << 16)
    w.cfl, w.mcfl = 0.0, 0.5
    w.q = w.q + 0.05 * w.h                            # a slow uniform flow sets the material dt
    s = _gpu_solver(w)
    assert s.spike is not None and s.cluster is None
    s.step()
    compare(w, s, [0], steps=1)
    s.run_steps(4)
    compare(w, s, [0], steps=5, tol=1e-10)
    d = s.diagnostics()
    assert d["rho_max"] > 50.0, d                     # decay r > 0.93 per row: no overlap of w <= 288 works
