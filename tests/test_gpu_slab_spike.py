"""GPU parity of the depth solve across slabs: every slab
runs tile-level SPIKE over its own tiles with the neighbouring slabs' rows from
the halo exchange, solves its separator system for Y and the spike columns V, W
of its two outer couplings, and all slabs solve the 2P end-separator system from
the all-gathered end values -- the exact solve of the whole domain's depth
system, with no overlap and no decay bound.  Against the single
domain on SPIKE (same equations, other tile cuts: round-off) and the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_STEP, _gather, compare, field_scales, oracle_run, rel_err
from tests.test_gpu_parity import gpu_solver as _gpu_solver

pytestmark = pytest.mark.gpu


def _hs():
    from paper_2510_07539_b200 import hsgn
    return hsgn


def spike_slabs(w, parts, mode=3):
    hs = _hs()
    solvers, edges = hs.slab_solvers(w, parts, align=4)
    for sv in solvers:
        sv.set_cluster(mode)
        assert sv.spike is not None, (sv.n, sv.spike)
    return solvers, edges


def single_spike(w):
    s = _gpu_solver(w)
    s.set_cluster(3)
    assert s.spike is not None
    return s


@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_slab_spike_group_equals_single_domain_and_oracle(parts, bc):
    hs = _hs()
    w = W.random_smooth(12000, 1, seed=parts, amp=0.08, bc=(bc, bc))
    w.filter_sigma = 0.25
    single = single_spike(w)
    solvers, _ = spike_slabs(w, parts)
    g = hs.Group(solvers)
    single.step()
    g.run_steps(1)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    refs, _ = oracle_run(w, [0], steps=1)
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc).dt(refs[0], w.cfl, w.mcfl)[0]
    S = field_scales(refs[0], float(w.lam[0]), dt)
    assert t[0] == t1[0]
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-13
    assert rel_err([h, q, K, Wf], refs[0], S) <= TOL_STEP
    g.run_steps(9)
    single.run_steps(9)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    assert abs(t[0] - t1[0]) <= 1e-13 * t1[0]
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-11
    compare(w, single, [0], steps=10, tol=1e-10)


def test_slab_spike_bathymetry_cfg5_recipe():
    hs = _hs()
    w = W.cfg5_workload(1 << 16)
    single = single_spike(w)
    solvers, _ = spike_slabs(w, 3)
    g = hs.Group(solvers)
    single.run_steps(5)
    g.run_steps(5)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    ref = [h1[0], q1[0], K1[0], W1[0]]
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), b=w.b).dt(ref, w.cfl, w.mcfl)[0]
    assert rel_err([h, q, K, Wf], ref, field_scales(ref, float(w.lam[0]), dt)) <= 1e-12
    assert abs(t[0] - t1[0]) <= 1e-13 * t1[0]
    compare(w, single, [0], steps=5, tol=1e-10)


def test_slab_spike_mcfl_only_large_rho_auto_mode():
    """material-CFL-only stepping (auto mode): the overlapped tiles cannot bound
    the decay, the slabs run SPIKE across slabs; the depth system couples over
    ~100 rows (rho ~ 10), far beyond the 3-cell stencil halo"""
    hs = _hs()
    w = W.random_smooth(8192, 1, seed=5, amp=0.3)
    w.cfl, w.mcfl = 0.0, 0.5                  # implied CFL_IMEX ~ 10
    single = single_spike(w)
    solvers, _ = spike_slabs(w, 4, mode=2)
    g = hs.Group(solvers)
    single.run_steps(3)
    g.run_steps(3)
    assert single.diagnostics()["rho_max"] > 5.0
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    ref = [h1[0], q1[0], K1[0], W1[0]]
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0])).dt(ref, w.cfl, w.mcfl)[0]
    # (round-off grows ~10x per step at this CFL_IMEX: 1.5e-11 in plain W after 3 steps)
    assert rel_err([h, q, K, Wf], ref, field_scales(ref, float(w.lam[0]), dt)) <= 1e-10
    compare(w, single, [0], steps=3, tol=1e-10)


@pytest.mark.parametrize("bc", ["periodic", "wall"])
def test_slab_spike_coupled_slabs_interface_system(bc):
    """8 slabs of 64 cells at an implied CFL_IMEX ~ 10: the depth system's
    inverse decays by only ~1e-9 over one slab, so the spike columns V, W and
    the 2P interface system carry real coupling (checked through
    hsgn_debug_copy); the result equals the single domain to round-off, and
    the oracle"""
    hs = _hs()
    w = W.random_smooth(512, 1, seed=5, amp=0.3, bc=(bc, bc))
    w.cfl, w.mcfl = 0.0, 0.3                  # implied CFL_IMEX 8-12
    w.filter_sigma = 0.25
    single = single_spike(w)
    solvers, _ = spike_slabs(w, 8, mode=2)
    assert all(sv.spike == (1, 64) for sv in solvers)
    g = hs.Group(solvers)
    single.step()
    g.run_steps(1)
    yvw = np.abs(solvers[3].debug_copy(1, 3))           # Y, V, W of slab 3 (one tile)
    assert yvw[1] > 1e-6 and yvw[2] > 1e-6, yvw           # (measured 1e-5 .. 5e-3, rho ~ 60-110)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    refs, _ = oracle_run(w, [0], steps=1)
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc).dt(refs[0], w.cfl, w.mcfl)[0]
    S = field_scales(refs[0], float(w.lam[0]), dt)
    assert t[0] == t1[0]
    # round-off only: at this CFL two builds of the oracle differ by 2e-13 (A17 floor)
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-12
    assert rel_err([h, q, K, Wf], refs[0], S) <= TOL_STEP
    g.run_steps(4)
    single.run_steps(4)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-11


def test_slab_spike_nccl_single_rank_ring():
    """the NCCL transport of the slab SPIKE stage with world = 1 (sends to and
    receives from itself, all-gather of one rank) == the single domain"""
    hs = _hs()
    w = W.random_smooth(8192, 1, seed=11, amp=0.08)
    w.filter_sigma = 0.25
    single = single_spike(w)
    (sv,), _ = spike_slabs(w, 1)
    sv.attach_nccl(hs.nccl_unique_id(), 0, 1)
    single.run_steps(10)
    sv.run_steps(10)
    (a, ta), (b, tb) = single.get_state(device=False), sv.get_state(device=False)
    ref = [f[0] for f in a]
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0])).dt(ref, w.cfl, w.mcfl)[0]
    assert rel_err([f[0] for f in b], ref, field_scales(ref, float(w.lam[0]), dt)) <= 1e-12
    assert abs(ta[0] - tb[0]) <= 1e-13 * ta[0]


def test_host_staged_slab_refuses_spike():
    hs = _hs()
    w = W.random_smooth(4096, 1, seed=3)
    solvers, _ = spike_slabs(w, 2)
    with pytest.raises(hs.HsgnError):
        solvers[0].slab_phase("stage1")
