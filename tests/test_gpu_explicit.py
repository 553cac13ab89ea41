"""GPU parity of the explicit hSGN scheme: the
CUDA explicit kernels through the C ABI against the oracle's explicit scheme
on the same seeded inputs; metric as in test_gpu_parity (A17)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, TOL_STEP, field_scales, gpu_solver, rel_err

pytestmark = pytest.mark.gpu

CFL_EX = 0.4          # the paper's explicit CFL


def _hsgn():
    from paper_2510_07539_b200 import hsgn
    return hsgn


def xsolver(w, stages=2, **kw):
    s = gpu_solver(w, **kw)
    s.set_params(w.g, w.lam, CFL_EX, 0.0)
    s.set_scheme("explicit", stages)
    return s


def xcompare(w, s, members, stages=2, steps=None, t_end=None, tol=TOL_STEP, order=2):
    (h, q, K, Wf), t = s.get_state(device=False)
    worst = 0.0
    for m in members:
        o = O.Oracle(w.n, w.dx, g=w.g, lam=float(w.lam[m]), bc=w.bc, order=order,
                     filter_sigma=w.filter_sigma)
        ref, tr, _ = o.explicit_run(w.state(m), cfl=CFL_EX, stages=stages, steps=steps,
                                    t_end=t_end)
        dt = o.dt(ref, CFL_EX, 0.0)[0]
        e = rel_err([h[m], q[m], K[m], Wf[m]], ref, field_scales(ref, float(w.lam[m]), dt, w.g))
        worst = max(worst, e)
        assert abs(t[m] - tr) <= max(tol, 1e-13) * max(1.0, abs(tr)), (m, t[m], tr)
    assert worst <= tol, worst
    return worst


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
@pytest.mark.parametrize("order,stages", [(2, 2), (1, 1), (2, 1)])
def test_explicit_one_step_ragged_tiles(bc, order, stages):
    w = W.random_smooth(3000, 3, seed=41, amp=0.08, bc=(bc, bc))
    s = xsolver(w, stages=stages, order=order)
    s.step()
    xcompare(w, s, range(3), stages=stages, steps=1, order=order)


@pytest.mark.parametrize("bc", ["periodic", "wall", "transmissive"])
def test_explicit_filter_runs(bc):
    w = W.random_smooth(2500, 2, seed=43, amp=0.05, bc=(bc, bc))
    w.filter_sigma = 0.25
    s = xsolver(w)
    s.run_steps(40)
    xcompare(w, s, range(2), steps=40, tol=1e-10)


def test_explicit_tiny_domains_wrap():
    for n, bc in ((4, "periodic"), (7, "periodic"), (5, "wall"), (9, "transmissive")):
        w = W.random_smooth(n, 2, seed=n, amp=0.02, bc=(bc, bc))
        s = xsolver(w)
        s.run_steps(3)
        xcompare(w, s, range(2), steps=3, tol=1e-10)


def test_explicit_dt_rule():
    w = W.random_smooth(1024, 3, seed=3, amp=0.1)
    s = xsolver(w)
    d = s.step(return_dt=True)
    for m in range(3):
        o = O.Oracle(w.n, w.dx, lam=float(w.lam[m]))
        ref, nu, _ = o.dt(w.state(m), CFL_EX, 0.0)
        assert abs(ref - CFL_EX * w.dx / nu) < 1e-15 * ref
        assert abs(d[m] - ref) <= 1e-14 * ref


def test_explicit_cfg1_soliton_run():
    """cfg1 soliton with the explicit scheme (filter on, A19/A22) to t = 2."""
    w = W.cfg1()
    s = xsolver(w)
    s.advance_to(2.0)
    (h, q, K, Wf), t = s.get_state(device=False)
    assert t[0] == 2.0
    xcompare(w, s, [0], t_end=2.0, tol=TOL_RUN)


def test_explicit_cfg3_subset_200_steps():
    w = W.cfg3(members=4)
    s = xsolver(w)
    s.run_steps(1)
    xcompare(w, s, range(4), steps=1)
    s.run_steps(199)
    xcompare(w, s, range(4), steps=200, tol=TOL_RUN)


@pytest.mark.parametrize("stages", [1, 2])
def test_explicit_launch_count(stages):
    w = W.random_smooth(512, 1, seed=1)
    s = xsolver(w, stages=stages)
    l0 = s.launches
    s.run_steps(40)
    s.sync()
    assert s.launches - l0 == 1 + (stages + 1) * 40


def test_explicit_refuses_bathymetry():
    hs = _hsgn()
    w = W.random_smooth(512, 1, seed=2, amp=0.05, bathy=0.05)
    s = xsolver(w)
    with pytest.raises(hs.HsgnError):
        s.run_steps(1)


def test_switching_back_to_si():
    """The scheme switch is per context: SI after explicit runs the SI step."""
    w = W.random_smooth(2048, 2, seed=5, amp=0.05)
    s = xsolver(w)
    s.set_scheme("si")
    s.set_params(w.g, w.lam, w.cfl, w.mcfl)
    s.step()
    (h, q, K, Wf), t = s.get_state(device=False)
    for m in range(2):
        o = O.Oracle(w.n, w.dx, lam=float(w.lam[m]), bc=w.bc, filter_sigma=w.filter_sigma)
        ref, *_ = o.run(w.state(m), cfl=w.cfl, mcfl=w.mcfl, steps=1)
        dt = o.dt(ref, w.cfl, w.mcfl)[0]
        assert rel_err([h[m], q[m], K[m], Wf[m]], ref, field_scales(ref, float(w.lam[m]), dt)) <= TOL_STEP
