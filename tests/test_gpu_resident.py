"""GPU parity of member-resident stepping (hsgn_run_resident, hsgn_multi.cuh):
K full SI-IMEX steps per launch with every member held in its cluster's
shared memory, against the oracle and against stepping on the cluster stage
kernels (same arithmetic up to rounding order)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, compare, field_scales, gpu_solver, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,bc", [(4096, "periodic"), (1000, "periodic"), (512, "periodic"), (3000, "wall"),
                                  (2048, "transmissive"), (8192, "periodic")])
def test_resident_matches_oracle_and_cluster_stepping(n, bc):
    w = W.random_smooth(n, 3, seed=n, amp=0.08, bc=(bc, bc))
    w.filter_sigma = 0.25
    a, b = gpu_solver(w), gpu_solver(w)
    b.set_cluster(1)
    a.run_resident(1)
    compare(w, a, range(3), steps=1, floor=True)
    a.run_resident(19)
    b.run_steps(20)
    compare(w, a, range(3), steps=20, tol=1e-10)
    (x, tx), (y, ty) = a.get_state(device=False), b.get_state(device=False)
    for m in range(3):
        ref = [f[m] for f in y]
        dt = O.Oracle(w.n, w.dx, lam=float(w.lam[m]), bc=w.bc).dt(ref, w.cfl, w.mcfl)[0]
        assert rel_err([f[m] for f in x], ref, field_scales(ref, float(w.lam[m]), dt)) <= 1e-12
    assert np.max(np.abs(tx - ty)) <= 1e-13 * np.max(ty)
    assert a.diagnostics()["steps"] == 20


def test_resident_bathymetry():
    w = W.random_smooth(4096, 2, seed=3, amp=0.05, bathy=0.08)
    w.filter_sigma = 0.25
    s = gpu_solver(w)
    s.run_resident(10)
    compare(w, s, range(2), steps=10, tol=1e-10)


def test_resident_cfg3_subset_200_steps_and_regular_stepping_after():
    w = W.cfg3(members=8)
    s = gpu_solver(w)
    s.run_resident(200)
    compare(w, s, range(8), steps=200, tol=TOL_RUN, floor=True)
    s.run_steps(5)                                    # the context continues on the regular kernels
    compare(w, s, range(8), steps=205, tol=TOL_RUN)


def test_resident_cfg1_to_t_end():
    w = W.cfg1()
    s = gpu_solver(w)
    s.run_resident(2000, t_end=w.t_end)
    (h, *_), t = s.get_state(device=False)
    assert t[0] == w.t_end
    compare(w, s, [0], t_end=w.t_end, tol=TOL_RUN, floor=True)


def test_resident_error_keeps_the_state():
    from paper_2510_07539_b200 import hsgn as hs
    w = W.random_smooth(512, 1, seed=4)
    s = hs.Solver(w.n, 1, w.x_min, w.x_max)
    s.set_params(9.81, w.lam, 2.0, 0.5, h_min=0.999)   # any h <= 0.999 is "dry"
    s.set_state(w.h.reshape(-1), w.q.reshape(-1), w.K.reshape(-1), w.W.reshape(-1))
    with pytest.raises(hs.HsgnError) as e:
        s.run_resident(5)
    assert e.value.name == "E_DRY"


@pytest.mark.slow
def test_resident_cfg3_full_size_sampled():
    """cfg3 at full size (4096 x 4096) in the bench's resident launch
    configuration (one launch of K steps, sub-record cfg3_resident); sampled
    members against the oracle after 1 and 200 steps"""
    from paper_2510_07539_b200 import hsgn as hs
    w = W.cfg3()
    s = hs.solver_for(w)
    sample = [0, 1, 777, 2048, 4095]
    s.run_resident(1)
    compare(w, s, sample, steps=1, floor=True)
    s.run_resident(199)
    assert s.diagnostics()["steps"] == 200
    compare(w, s, sample[:3], steps=200, tol=TOL_RUN, floor=True)
