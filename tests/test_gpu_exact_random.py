"""Seeded random cases for the exact depth-solve organisations (DESIGN.md
sections 6 and 8): cluster kernels, tile-level SPIKE, SPIKE across slabs, and
the member-resident kernel, each against the oracle (metric A17) after one and
after five steps on ragged sizes, all boundary kinds, orders 1 / 2, the paper's
and the Euler tableau, bathymetry, filter, and material-CFL-only stepping."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import _gather, compare, field_scales, oracle_run, rel_err
from tests.test_gpu_parity import gpu_solver as _gpu_solver

pytestmark = pytest.mark.gpu


def _hs():
    from paper_2510_07539_b200 import hsgn
    return hsgn


def _case(seed, n_lo, n_hi, mult=4):
    """a random workload (n a multiple of `mult`), its solver keywords and oracle keywords"""
    hs = _hs()
    rng = np.random.default_rng(seed)
    n = mult * int(rng.integers(n_lo // mult, n_hi // mult))
    members = int(rng.integers(1, 3))
    bc = ["periodic", "wall", "transmissive"][int(rng.integers(0, 3))]
    bathy = float(rng.choice([0.0, 0.05]))
    w = W.random_smooth(n, members, seed=int(rng.integers(1 << 30)), amp=float(rng.uniform(0.02, 0.12)),
                        bc=(bc, bc), bathy=bathy, lam_range=(10 ** rng.uniform(1.5, 2.5), 10 ** rng.uniform(3, 4.2)))
    w.filter_sigma = float(rng.choice([0.0, 0.25]))
    if rng.random() < 0.3:                          # material-CFL-only stepping
        w.cfl, w.mcfl = 0.0, 0.3
    kw, okw = {"order": int(rng.integers(1, 3))}, {}
    okw["order"] = kw["order"]
    if rng.random() < 0.3:
        kw["tableau"] = hs.euler_tableau()
        okw["tableau"] = O.euler_tableau()
    if w.cfl == 0.0:
        # large implied CFL_IMEX: keep the case only where the scheme itself stays
        # coercive for the 5 steps (the oracle decides; else CFL_IMEX 2)
        try:
            oracle_run(w, range(w.members), steps=5, **okw)
        except O.OracleError:
            w.cfl, w.mcfl = 2.0, 0.5
    return w, kw, okw


def _check(w, s, okw, members):
    s.step()
    compare(w, s, members, steps=1, floor=True, **okw)
    s.run_steps(4)
    compare(w, s, members, steps=5, tol=1e-10, **okw)


@pytest.mark.parametrize("case", range(10))
def test_random_cluster(case):
    w, kw, okw = _case(9100 + case, 8, 8192)
    s = _gpu_solver(w, **kw)
    s.set_cluster(1)
    assert s.cluster is not None, (w.n, w.bc)
    _check(w, s, okw, range(w.members))


@pytest.mark.parametrize("case", range(10))
def test_random_spike(case):
    w, kw, okw = _case(9200 + case, 8, 40000)
    s = _gpu_solver(w, **kw)
    s.set_cluster(3)
    assert s.spike is not None, (w.n, w.bc)
    _check(w, s, okw, range(w.members))


@pytest.mark.parametrize("case", range(8))
def test_random_slab_spike(case):
    """a one-member random case split into 2..5 slabs (group transport) on
    SPIKE across slabs: equal to the single domain on SPIKE (round-off) and the
    oracle"""
    hs = _hs()
    w, kw, okw = _case(9300 + case, 2000, 30000)
    rng = np.random.default_rng(case)
    parts = int(rng.integers(2, 6))
    if w.members > 1:
        w = W.Workload(w.name, w.n, 1, w.x_min, w.x_max, w.bc, w.lam[:1], w.h[:1], w.q[:1], w.K[:1], w.W[:1],
                       b=w.b, cfl=w.cfl, mcfl=w.mcfl, filter_sigma=w.filter_sigma)
    single = _gpu_solver(w, **kw)
    single.set_cluster(3)
    solvers, _ = hs.slab_solvers(w, parts, align=4, order=kw["order"])
    for sv in solvers:
        if "tableau" in kw:
            sv.set_tableau(kw["tableau"])
        sv.set_cluster(3)
        assert sv.spike is not None
    g = hs.Group(solvers)
    single.step()
    g.run_steps(1)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    refs, _ = oracle_run(w, [0], steps=1, **okw)
    dt = O.Oracle(w.n, w.dx, lam=float(w.lam[0]), bc=w.bc, b=w.b).dt(refs[0], w.cfl, w.mcfl)[0]
    S = field_scales(refs[0], float(w.lam[0]), dt)
    assert t[0] == t1[0]
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-12
    compare(w, single, [0], steps=1, floor=True, **okw)
    g.run_steps(4)
    single.run_steps(4)
    (h, q, K, Wf), t = _gather(solvers)
    (h1, q1, K1, W1), t1 = single.get_state(device=False)
    assert abs(t[0] - t1[0]) <= 1e-13 * t1[0]
    assert rel_err([h, q, K, Wf], [h1[0], q1[0], K1[0], W1[0]], S) <= 1e-10


@pytest.mark.parametrize("case", range(8))
def test_random_resident(case):
    """run_resident (one launch of 5 steps) == the oracle; 2-stage tableau only"""
    w, kw, okw = _case(9400 + case, 8, 8192)
    kw.pop("tableau", None)
    okw.pop("tableau", None)
    s = _gpu_solver(w, **kw)
    s.set_cluster(1)
    assert s.cluster is not None
    s.run_resident(1)
    compare(w, s, range(w.members), steps=1, floor=True, **okw)
    s.run_resident(4)
    compare(w, s, range(w.members), steps=5, tol=1e-10, **okw)
