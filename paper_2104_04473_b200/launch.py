"""Process-group plumbing shared by bench.py and the multi-process tests.

torch.distributed is used only to bootstrap: read RANK / WORLD_SIZE /
LOCAL_RANK from the launcher, hand rank 0's NCCL unique id to every rank, and
reduce timings (max over ranks).  All collectives of the hot path run inside
libmp.so on its own NCCL communicators and IPC channels.
"""
import os


def env_ranks():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 if absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_bytes(blob_or_none, rank, world):
    """Broadcast rank 0's bytes (e.g. the NCCL unique id) to every rank."""
    if world == 1:
        return blob_or_none
    import torch.distributed as dist
    obj = [blob_or_none if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(x, world, device=None):
    """Max of a float over all ranks (the bench's timing rule)."""
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def tp_pp_of(rank, t, p):
    """Grid coordinates of a rank: rank = (dp * p + pp) * t + tp."""
    return rank % t, (rank // t) % p, rank // (t * p)
