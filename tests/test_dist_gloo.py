"""Multi-process host logic on CPU with gloo (world_size 2): sharding arithmetic,
the unique-id bootstrap and max-over-ranks timing used by bench.py and by slab
contexts (paper_2510_07539_b200/dist.py)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_07539_b200 import dist as D
    out = {}
    out["slab"] = D.slab_range(1 << 28, rank, world)
    out["shard"] = D.shard_members(4096 * world, rank, world)
    payload = bytes(range(128)) if rank == 0 else None
    out["uid"] = D.broadcast_bytes(payload, 128)
    out["max"] = D.max_over_ranks([float(rank), 10.0 - rank])
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, out))


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # slabs tile [0, 2^28) without gaps or overlap
    edges = sorted(res[r]["slab"] for r in range(world))
    assert edges[0][0] == 0 and edges[-1][1] == 1 << 28
    assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
    # ensemble shards: 4096 members per rank, disjoint, covering
    assert [res[r]["shard"] for r in range(world)] == [(4096 * r, 4096) for r in range(world)]
    # the 128-byte unique id reaches every rank intact
    assert all(res[r]["uid"] == bytes(range(128)) for r in range(world))
    # element-wise max over ranks
    assert all(res[r]["max"] == [float(world - 1), 10.0] for r in range(world))


def test_slab_edges_local():
    from paper_2510_07539_b200 import dist as D
    for n in (4096, 1 << 20, 1000003):
        for world in (1, 2, 3, 8):
            e = D.slab_edges(n, world)
            assert e[0] == 0 and e[-1] == n
            sizes = [b - a for a, b in zip(e, e[1:])]
            assert max(sizes) - min(sizes) <= 1


def _ring_worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_07539_b200 import dist as D
    H = 5
    bnd = np.concatenate([np.full(H, 100.0 * rank + 1), np.full(H, 100.0 * rank + 2)])   # [left | right]
    halo = D._ring_exchange(bnd, rank, world)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, halo.tolist()))


@pytest.mark.parametrize("world", [2, 3])
def test_host_staged_ring_exchange(world):
    """host-staged slab transport: rank r's [left halo | right halo] is
    [right boundary of r-1 | left boundary of r+1] on the periodic ring"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ring_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        left, right = (r - 1) % world, (r + 1) % world
        assert res[r] == [100.0 * left + 2] * 5 + [100.0 * right + 1] * 5
