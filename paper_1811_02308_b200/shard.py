"""Multi-GPU host logic: the fast adaptive bilateral filter partitions into
independent problems (frames of a batch), so N GPUs each
filter their own frames with no data-path collective.  One process per GPU
(torchrun); the only collective is the max-over-ranks of the timed region
(plain torch.distributed, NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def frame_shard(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of frames owned by ``rank``: (first, count).  The first
    ``batch % world`` ranks take one extra frame; counts differ by at most 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if batch < 0:
        raise ValueError("batch < 0")
    base, extra = divmod(batch, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_frames(local, batch: int, world: int, rank: int):
    """Reassemble a sharded batch on every rank: ``local`` holds this rank's
    frames (first axis, in frame_shard order, host arrays); returns the whole
    (batch, ...) array.  The only data-path collective of the sharded path,
    used when a caller wants the frames back in one place (the bench does not:
    each rank keeps its own output)."""
    import numpy as np
    import torch.distributed as dist

    first, n = frame_shard(batch, world, rank)
    if len(local) != n:
        raise ValueError(f"rank {rank} holds {len(local)} frames, its shard has {n}")
    if world == 1 or not (dist.is_available() and dist.is_initialized()):
        return np.asarray(local)
    parts = [None] * world
    dist.all_gather_object(parts, (first, np.asarray(local)))
    return np.concatenate([p for _, p in sorted(parts, key=lambda t: t[0]) if len(p)], axis=0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the device time of the timed region) over the
    process group; identity without an initialised group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(pixels_per_rank: list[int] | int, steps: int, seconds: float, world: int = 1) -> float:
    """Whole-job throughput (Mpix/s): every rank's pixels over the max-over-ranks
    time.  ``pixels_per_rank`` is a list (per rank) or one count for all."""
    total = sum(pixels_per_rank) if isinstance(pixels_per_rank, list) else pixels_per_rank * world
    return total * steps / seconds / 1e6
