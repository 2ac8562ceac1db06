"""Host-side slab-decomposition logic shared by bench.py and the tests
(SPEC.md:479-548 parallel runtime; the device side is csrc/dist.cu).

* `slab`: x1 planes owned by a rank (equal contiguous slabs, like slab_of in
  csrc/ctx.cu).
* `halo_exchange`: the ghost-plane protocol of csrc/dist.cu (halo_exchange)
  written against torch.distributed, so the message ordering -- the part that
  matters when both ring neighbours are the same peer (p = 2) -- is tested on
  CPU with gloo.
* `fold_plane_partials`: the plane-ordered fp64 fold that makes every
  reduction bitwise independent of the rank count (field.hpp:143-155).
* `init_from_env`: one process per GPU under torchrun; NCCL communicator of
  the device library bootstrapped from a unique id broadcast over
  torch.distributed.
"""
from __future__ import annotations

import os


def slab(n1: int, rank: int, nranks: int):
    if n1 % nranks:
        raise ValueError("slab layout infeasible: n1 must be divisible by the rank count")
    n1l = n1 // nranks
    return n1l, rank * n1l


def neighbours(rank: int, nranks: int):
    return (rank - 1) % nranks, (rank + 1) % nranks


def halo_exchange(local, G: int, group=None):
    """Return (lo, hi): the G planes below / above this rank's slab
    (periodic ring). Same send/recv order as csrc/dist.cu: per peer, the
    message landing in the peer's lo goes first."""
    import torch
    import torch.distributed as dist
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    if G > local.shape[0]:
        raise ValueError("ghost width exceeds the slab width")
    prev, nxt = neighbours(rank, p)
    lo = torch.empty_like(local[:G])
    hi = torch.empty_like(local[:G])
    ops = [dist.P2POp(dist.isend, local[-G:].contiguous(), nxt, group),
           dist.P2POp(dist.isend, local[:G].contiguous(), prev, group),
           dist.P2POp(dist.irecv, lo, prev, group),
           dist.P2POp(dist.irecv, hi, nxt, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    return lo, hi


def plane_partials(local):
    """fp64 per-x1-plane sums of a slab (one value per plane)."""
    return local.double().reshape(local.shape[0], -1).sum(dim=1)


def fold_plane_partials(partials):
    """Fold per-plane partials in global plane order (left to right)."""
    total = 0.0
    for x in partials.tolist():
        total += x
    return total


def init_from_env():
    """(ctx, rank, world, local_rank) for the current torchrun process."""
    import torch
    import torch.distributed as dist
    from .engine import Context
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world == 1:
        return Context(local), 0, 1, local
    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    obj = [Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Context(local, rank, world, obj[0]), rank, world, local
