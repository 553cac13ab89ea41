"""Multi-GPU plumbing (torch.distributed): sharding arithmetic, the NCCL
unique-id bootstrap for slab contexts, and max-over-ranks timing.  Pure host
logic; the data path (halo exchange, dt all-reduce) runs inside libhsgn.so
(include/hsgn.h: hsgn_attach_nccl), or -- host-staged transport -- through
the process group's own collectives between the library's step phases
(host_staged_step; gloo).  Covered by tests/test_dist_gloo.py on CPU
(world_size 2, gloo)."""
from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def slab_edges(n: int, world: int) -> list[int]:
    """Contiguous slabs of a domain of n cells; sizes differ by at most one."""
    return [(i * n) // world for i in range(world + 1)]


def slab_range(n: int, rank: int, world: int) -> tuple[int, int]:
    e = slab_edges(n, world)
    return e[rank], e[rank + 1]


def shard_members(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of an ensemble of `total` members for this rank."""
    a, b = slab_range(total, rank, world)
    return a, b - a


def _device():
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def broadcast_bytes(data: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast a fixed-size byte string from `src` (e.g. a 128-B ncclUniqueId)."""
    t = torch.zeros(nbytes, dtype=torch.uint8, device=_device())
    if dist.get_rank() == src:
        assert data is not None and len(data) == nbytes
        t.copy_(torch.frombuffer(bytearray(data), dtype=torch.uint8))
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def max_over_ranks(values):
    """Element-wise max over ranks of a list of floats (timings are max-reduced)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=_device())
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu().tolist()]


def _ring_exchange(bnd, rank: int, world: int, group=None):
    """[left boundary | right boundary] of every rank -> this rank's
    [left halo | right halo] = [left neighbour's right boundary | right
    neighbour's left boundary] (ring; an all_gather, any world size)."""
    half = bnd.size // 2
    t = torch.from_numpy(bnd.copy())
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    left, right = parts[(rank - 1) % world].numpy(), parts[(rank + 1) % world].numpy()
    return np.concatenate([left[half:], right[:half]])


def host_staged_exchange_b(solver, rank: int, world: int, group=None):
    """Static bathymetry halos of a host-staged slab (once, before stepping)."""
    solver.slab_put("b", _ring_exchange(solver.slab_get("b"), rank, world, group))


def host_staged_step(solver, rank: int, world: int, group=None, stages: int = 2):
    """One slab step through the host-staged transport (include/hsgn.h): the
    dt maxima max-reduced and the U^n / U1 halos exchanged with the process
    group's collectives (gloo on CPU tensors), the stages on the GPU."""
    mx = solver.slab_get("maxima").view(np.int64)        # non-negative doubles: int64 order
    t = torch.from_numpy(mx.copy())
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    solver.slab_put("maxima", t.numpy().view(np.uint64))
    solver.slab_phase("dt")
    solver.slab_put("un", _ring_exchange(solver.slab_get("un"), rank, world, group))
    solver.slab_phase("stage1")
    if stages == 2:
        solver.slab_put("u1", _ring_exchange(solver.slab_get("u1"), rank, world, group))
        solver.slab_phase("stage2")
    solver.slab_phase("commit")


def attach_slab(solver, rank: int, world: int):
    """NCCL bootstrap of a slab context: rank 0 creates the unique id, every
    rank receives it through torch.distributed and joins the ring."""
    from . import hsgn
    uid = hsgn.nccl_unique_id() if rank == 0 else None
    uid = broadcast_bytes(uid, 128, src=0)
    solver.attach_nccl(uid, rank, world)
