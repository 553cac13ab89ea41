"""GPU parity of the classical SGN scheme: the
CUDA sgn_kernel through the C ABI against the oracle's SGN scheme on the same
seeded inputs.  Metric: max_i |f_gpu - f_ref| / max(max|f_ref|, sqrt(g h_max) h_max)
for q and / max|h| for h (A17); K and W are carried unchanged."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, TOL_STEP, gpu_solver

pytestmark = pytest.mark.gpu

CFL_SGN = 0.9


def _hsgn():
    from paper_2510_07539_b200 import hsgn
    return hsgn


def ssolver(w, stages=2, **kw):
    hs = _hsgn()
    order = kw.pop("order", 2)
    s = hs.Solver(w.n, w.members, w.x_min, w.x_max, bc=w.bc, order=order, **kw)
    s.set_params(w.g, w.lam, CFL_SGN, 0.0)
    if w.b is not None:
        s.set_bathymetry(w.b)
    s.set_scheme("sgn", stages)
    s.set_state(w.h.reshape(-1), w.q.reshape(-1), w.K.reshape(-1), w.W.reshape(-1))
    return s


def scompare(w, s, members, stages=2, steps=None, t_end=None, tol=TOL_STEP, order=2):
    (h, q, K, Wf), t = s.get_state(device=False)
    worst = 0.0
    for m in members:
        o = O.Oracle(w.n, w.dx, g=w.g, bc=w.bc, order=order, b=w.b)
        U0 = w.state(m)
        ref, tr, _ = o.sgn_run(U0, cfl=CFL_SGN, stages=stages, steps=steps, t_end=t_end)
        hm = np.max(np.abs(ref[0]))
        Sq = max(np.max(np.abs(ref[1])), np.sqrt(w.g * hm) * hm)
        e = max(np.max(np.abs(h[m] - ref[0])) / hm, np.max(np.abs(q[m] - ref[1])) / Sq)
        assert np.array_equal(K[m], U0[2]) and np.array_equal(Wf[m], U0[3])   # carried
        worst = max(worst, e)
        assert abs(t[m] - tr) <= max(tol, 1e-13) * max(1.0, abs(tr)), (m, t[m], tr)
    assert worst <= tol, worst
    return worst


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 1), (2, 1)])
def test_sgn_one_step_ragged_tiles(bc, order, stages):
    w = W.random_smooth(5000, 3, seed=51, amp=0.08, bc=(bc, bc))
    w.filter_sigma = 0.0
    s = ssolver(w, stages=stages, order=order)
    s.step()
    scompare(w, s, range(3), stages=stages, steps=1, order=order)


def test_sgn_runs_walls_and_periodic():
    for bc in ("periodic", "wall", "transmissive"):
        w = W.random_smooth(3000, 2, seed=53, amp=0.05, bc=(bc, bc))
        w.filter_sigma = 0.0
        s = ssolver(w)
        s.run_steps(40)
        scompare(w, s, range(2), steps=40, tol=1e-10)


def test_sgn_tiny_domains_wrap():
    for n, bc in ((4, "periodic"), (7, "periodic"), (5, "wall"), (9, "transmissive")):
        w = W.random_smooth(n, 2, seed=n, amp=0.02, bc=(bc, bc), dx=0.5)
        w.filter_sigma = 0.0
        s = ssolver(w)
        s.run_steps(3)
        scompare(w, s, range(2), steps=3, tol=1e-10)


def test_sgn_dt_rule():
    w = W.random_smooth(2048, 3, seed=3, amp=0.1)
    w.filter_sigma = 0.0
    s = ssolver(w)
    d = s.step(return_dt=True)
    for m in range(3):
        o = O.Oracle(w.n, w.dx)
        ref = o.sgn_dt(w.state(m), CFL_SGN)
        assert abs(d[m] - ref) <= 1e-14 * ref


def test_sgn_cfg1_soliton_run():
    """cfg1 soliton with the classical SGN scheme to t = 2 (an exact SGN solution)."""
    w = W.cfg1()
    w.filter_sigma = 0.0
    s = ssolver(w)
    s.advance_to(2.0)
    (h, q, K, Wf), t = s.get_state(device=False)
    assert t[0] == 2.0
    scompare(w, s, [0], t_end=2.0, tol=TOL_RUN)
    he, _ = W.soliton_exact(w.x(), 2.0, 1.0, 0.2, -50.0, L=200.0)
    assert np.sum(np.abs(h[0] - he)) / np.sum(np.abs(h[0])) < 1e-3


def test_sgn_cfg3_subset_200_steps():
    w = W.cfg3(members=4)
    w.filter_sigma = 0.0
    s = ssolver(w)
    s.run_steps(1)
    scompare(w, s, range(4), steps=1)
    s.run_steps(199)
    scompare(w, s, range(4), steps=200, tol=TOL_RUN)


@pytest.mark.parametrize("stages", [1, 2])
def test_sgn_launch_count(stages):
    w = W.random_smooth(512, 1, seed=1)
    w.filter_sigma = 0.0
    s = ssolver(w, stages=stages)
    l0 = s.launches
    s.run_steps(40)
    s.sync()
    assert s.launches - l0 == 1 + (stages + 1) * 40


def test_sgn_refuses_filter_and_too_fine_grids():
    hs = _hsgn()
    w = W.random_smooth(1024, 1, seed=2, amp=0.05)
    w.filter_sigma = 0.0
    s = ssolver(w)
    s.set_filter(0.25)
    with pytest.raises(hs.HsgnError):
        s.run_steps(1)
    fine = W.random_smooth(20000, 1, seed=2, amp=0.05, dx=0.005)   # h/dx = 200
    with pytest.raises(hs.HsgnError):
        ssolver(fine)


# --------------------------------------------------------------------------
# bathymetric SGN (reading A26)
@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 1)])
def test_sgnb_one_step_ragged_tiles(bc, order, stages):
    w = W.random_smooth(5000, 3, seed=57, amp=0.06, bc=(bc, bc), bathy=0.08)
    w.filter_sigma = 0.0
    s = ssolver(w, stages=stages, order=order)
    assert s.geometry.tiles_per_member > 1
    s.step()
    scompare(w, s, range(3), stages=stages, steps=1, order=order)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_sgnb_runs(bc):
    w = W.random_smooth(3000, 2, seed=59, amp=0.05, bc=(bc, bc), bathy=0.06)
    w.filter_sigma = 0.0
    s = ssolver(w)
    s.run_steps(40)
    scompare(w, s, range(2), steps=40, tol=1e-10)


def test_sgnb_zero_bathymetry_is_the_flat_path():
    w = W.random_smooth(2048, 2, seed=61, amp=0.05)
    w.filter_sigma = 0.0
    a = ssolver(w)
    w.b = np.zeros(w.n)
    b = ssolver(w)
    a.run_steps(10)
    b.run_steps(10)
    (x, _), (y, _) = a.get_state(device=False), b.get_state(device=False)
    for f, g in zip(x, y):
        assert np.max(np.abs(f - g)) <= 1e-13 * max(1.0, np.max(np.abs(f)))


def test_sgnb_lake_at_rest_small_drift():
    """zeta = const, u = 0 over bathymetry: phi = 0 and only the O(dx^2) residual
    of the centred hydrostatic source moves water (oracle pin
    test_sgnb_lake_at_rest_second_order); the GPU equals the oracle on it."""
    w = W.lake_at_rest(2000, 0.0)
    w.filter_sigma = 0.0
    s = ssolver(w)
    s.run_steps(50)
    scompare(w, s, [0], steps=50, tol=1e-10)
    (h, q, K, Wf), t = s.get_state(device=False)
    assert np.max(np.abs(q[0])) < 1e-3
