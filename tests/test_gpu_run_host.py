"""hsgn_run_host (include/hsgn.h): a whole ensemble job from host memory,
pipelined over member chunks.  Members are independent, so every member's
result must be bitwise the one of hsgn_set_state + hsgn_run_steps +
hsgn_get_state (itself parity-tested against the oracle in test_gpu_parity);
two members are also compared with the oracle directly."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_07539_b200 import workloads as W
from tests.test_gpu_parity import TOL_RUN, field_scales, gpu_solver, rel_err

pytestmark = pytest.mark.gpu


def _hsgn():
    from paper_2510_07539_b200 import hsgn
    return hsgn


def plain(w, steps, **kw):
    s = gpu_solver(w, **kw)
    s.run_steps(steps)
    return s.get_state(device=False)


def host_inputs(w):
    return [np.ascontiguousarray(f.reshape(-1)) for f in (w.h, w.q, w.K, w.W)]


def assert_same(a, b):
    (x, tx), (y, ty) = a, b
    for f, g in zip(x, y):
        assert np.array_equal(f, g)
    assert np.array_equal(tx, ty)


@pytest.mark.parametrize("chunks", [1, 3, 8, 40])
def test_run_host_bitwise_equals_plain_path(chunks):
    w = W.random_smooth(3000, 10, seed=81, amp=0.08)
    ref = plain(w, 25, tile_cells=700)
    s = gpu_solver(w, tile_cells=700)
    got = s.run_host(*host_inputs(w), 25, chunks=chunks)
    assert_same(got, ref)


@pytest.mark.parametrize("bc", ["wall", "transmissive"])
def test_run_host_bathymetry_filter_walls(bc):
    w = W.random_smooth(2048, 5, seed=83, amp=0.05, bc=(bc, bc), bathy=0.08)
    w.filter_sigma = 0.25
    ref = plain(w, 20, tile_cells=512)
    s = gpu_solver(w, tile_cells=512)
    assert_same(s.run_host(*host_inputs(w), 20, chunks=2), ref)


def test_run_host_relaxation_zones_and_variants():
    w = W.cfg4(n=1 << 14)
    ref = plain(w, 30)
    s = gpu_solver(w)
    assert_same(s.run_host(*host_inputs(w), 30, chunks=4), ref)
    # explicit scheme, well-balanced form, Picard passes: same settings reach the chunks
    v = W.random_smooth(1024, 6, seed=85, amp=0.05)
    for setup in (lambda s: (s.set_params(v.g, v.lam, 0.4, 0.0), s.set_scheme("explicit")),
                  lambda s: s.set_well_balanced(True), lambda s: s.set_picard(1)):
        a = gpu_solver(v)
        setup(a)
        a.run_steps(12)
        ref = a.get_state(device=False)
        b = gpu_solver(v)
        setup(b)
        assert_same(b.run_host(*host_inputs(v), 12, chunks=3), ref)


def test_run_host_matches_oracle_and_reruns():
    w = W.cfg3(members=6, n=2048)
    s = gpu_solver(w)
    inp = host_inputs(w)
    (h, q, K, Wf), t = s.run_host(*inp, 60, chunks=4)
    for m in (0, 5):
        o = O.Oracle(w.n, w.dx, lam=float(w.lam[m]), bc=w.bc, filter_sigma=w.filter_sigma)
        ref, tr, _, _ = o.run(w.state(m), cfl=w.cfl, mcfl=w.mcfl, steps=60)
        dt = o.dt(ref, w.cfl, w.mcfl)[0]
        assert rel_err([h[m], q[m], K[m], Wf[m]], ref, field_scales(ref, float(w.lam[m]), dt)) <= TOL_RUN
        assert abs(t[m] - tr) <= 1e-12 * tr
    again = s.run_host(*inp, 60, chunks=4)           # views reused, same result
    assert_same(again, ((h, q, K, Wf), t))
    s.set_filter(0.0)                                # a setter rebuilds the chunk views
    w.filter_sigma = 0.0
    assert_same(s.run_host(*inp, 10, chunks=4), plain(w, 10))


def test_run_host_pinned_torch_buffers():
    import torch
    w = W.random_smooth(4096, 8, seed=87, amp=0.05)
    ref = plain(w, 18)
    s = gpu_solver(w)
    inp = [torch.from_numpy(a).pin_memory() for a in host_inputs(w)]
    out = [torch.empty(w.members * w.n, dtype=torch.float64).pin_memory() for _ in range(4)]
    _, t = s.run_host(*inp, 18, out=out, chunks=4)
    assert_same(([o.numpy().reshape(w.members, w.n) for o in out], t), ref)


def test_run_host_error_in_one_chunk():
    """A coercivity failure (eta/h = 0.2 at lam = 1000, as in
    test_coercivity_violation_reported) in member 2 stops its chunk at its last
    committed state (the initial one); the other chunks complete."""
    hs = _hsgn()
    w = W.random_smooth(256, 4, seed=89, amp=0.05, dx=0.1)
    w.lam[:] = 1000.0
    w.K[2] = 0.2 * w.h[2] ** 2
    s = gpu_solver(w)
    with pytest.raises(hs.HsgnError) as e:
        s.run_host(*host_inputs(w), 5, chunks=4)
    assert e.value.name == "E_COERCIVITY"
    import ctypes as C
    out = [np.empty((w.members, w.n)) for _ in range(4)]
    t = np.empty(w.members)
    st = s.L.hsgn_run_host(s.ctx, *[C.c_void_p(a.ctypes.data) for a in host_inputs(w)], 0.0, 5,
                           *[C.c_void_p(a.ctypes.data) for a in out], C.c_void_p(t.ctypes.data), 4)
    assert st != 0
    assert np.array_equal(out[0][2], w.h[2]) and np.array_equal(out[2][2], w.K[2]) and t[2] == 0.0
    good = w.subset([0, 1, 3])
    ref, tr = plain(good, 5)
    for i, m in enumerate((0, 1, 3)):
        for f in range(4):
            assert np.array_equal(out[f][m], ref[f][i])
        assert t[m] == tr[i]


def test_run_host_state_and_refusals():
    hs = _hsgn()
    w = W.random_smooth(1024, 2, seed=91, amp=0.05)
    s = gpu_solver(w)
    s.run_host(*host_inputs(w), 3, chunks=2)
    with pytest.raises(hs.HsgnError):          # no state after run_host
        s.run_steps(1)
    s.set_state(*host_inputs(w))
    s.run_steps(1)
    s.sync()
    g = gpu_solver(w)
    g.set_params(w.g, w.lam, 0.9, 0.0)
    g.set_scheme("sgn")
    with pytest.raises(hs.HsgnError):
        g.run_host(*host_inputs(w), 3)
