"""Multi-GPU host plumbing (one process per GPU, launched by torch.distributed.run).

The process group only carries the 128-byte NCCL id and the benchmark's
max-over-ranks timing; the counting path's one exchange step (the u64
allreduce of the outputs) runs inside libbf on its own NCCL communicator.
"""
from __future__ import annotations


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) from `src` over the default group."""
    import torch.distributed as dist
    box = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (device timing rule)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def nccl_comm_for_group(device_index: int):
    """Create libbf's NCCL communicator for this rank: rank 0 makes the id, the
    process group broadcasts it, every rank joins."""
    import torch.distributed as dist
    from . import bf
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = broadcast_bytes(bf.bf_nccl_unique_id() if rank == 0 else None)
    return bf.bf_nccl_comm_create(uid, rank, world, device_index)


def rank_share(rank: int, world: int, t0: int, t1: int) -> list[int]:
    """Indices of [t0, t1) this rank processes (libbf's own deal function)."""
    from . import bf
    out, q = [], 0
    while True:
        i = bf.bf_deal_index(q, rank, world, t0, t1)
        if i >= t1:
            return out
        out.append(i)
        q += 1
