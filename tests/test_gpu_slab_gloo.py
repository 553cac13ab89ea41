"""Multi-rank slab data path on one GPU: two processes, each one slab of a
periodic domain (cfg5 recipe with bathymetry), stepping through the
host-staged transport (include/hsgn.h hsgn_slab_get / put / phase) with the
dt maxima max-reduced and the halos exchanged by gloo collectives.  The
ranks' kernels never wait on each other (the exchange is on the host).  The
gathered state must equal the single-domain solve to round-off."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_07539_b200 import workloads as W

pytestmark = pytest.mark.gpu

N_CELLS, STEPS = 1 << 16, 10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slab_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2510_07539_b200 import dist as D
        from paper_2510_07539_b200 import hsgn
        w = W.cfg5_workload(N_CELLS)
        a, b = D.slab_range(w.n, rank, world)
        sv = hsgn.Solver(b - a, 1, w.x_min + a * w.dx, w.x_min + b * w.dx, bc=("halo", "halo"))
        sv.set_params(w.g, w.lam, w.cfl, w.mcfl)
        sv.set_bathymetry(np.ascontiguousarray(w.b[a:b]))
        sv.set_filter(w.filter_sigma)
        sv.set_state(*[np.ascontiguousarray(f[0, a:b]) for f in (w.h, w.q, w.K, w.W)])
        D.host_staged_exchange_b(sv, rank, world)
        out = []
        for k in range(STEPS):
            D.host_staged_step(sv, rank, world)
            if k in (0, STEPS - 1):
                (h, q_, K, Wf), t = sv.get_state(device=False)
                out.append(([h[0], q_[0], K[0], Wf[0]], float(t[0])))
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None))
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_host_staged_slabs_equal_single_domain():
    from paper_2510_07539_b200 import hsgn
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, out, _ = q.get(timeout=600)
        assert not isinstance(out, str), out
        res[r] = out
    for p in ps:
        p.join(timeout=120)
    w = W.cfg5_workload(N_CELLS)
    # (1) the same slab decomposition in one process (loopback group transport):
    #     identical arithmetic and tile cuts -> bitwise equal
    solvers, _ = hsgn.slab_solvers(w, world)
    g = hsgn.Group(solvers)
    single = hsgn.solver_for(w)
    for i, nst in enumerate((1, STEPS - 1)):
        g.run_steps(nst)
        single.run_steps(nst)
        got = [np.concatenate([res[r][i][0][k] for r in range(world)]) for k in range(4)]
        assert res[0][i][1] == res[1][i][1]                      # one global dt per step
        outs = [sv.get_state(device=False) for sv in solvers]
        grp = [np.concatenate([o[0][k][0] for o in outs]) for k in range(4)]
        for a_, b_ in zip(got, grp):
            assert np.array_equal(a_, b_)
        assert outs[0][1][0] == res[0][i][1]
        # (2) the single domain (different tile cuts: round-off apart)
        (h, q_, K, Wf), t = single.get_state(device=False)
        ref = [h[0], q_[0], K[0], Wf[0]]
        assert abs(res[0][i][1] - t[0]) <= 1e-13 * t[0]
        lam, dt = float(w.lam[0]), single.diagnostics()["dt_last_max"]
        scales = [np.max(np.abs(ref[0])), max(np.max(np.abs(ref[1])), np.sqrt(9.81 * ref[0].max()) * ref[0].max()),
                  np.max(np.abs(ref[2])), max(np.max(np.abs(ref[3])), lam * dt)]
        err = max(np.max(np.abs(x - y)) / sc for x, y, sc in zip(got, ref, scales))
        assert err <= (1e-13 if i == 0 else 1e-12), (i, err)
