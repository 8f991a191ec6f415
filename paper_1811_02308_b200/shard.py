"""Multi-GPU host logic: the fast adaptive bilateral filter partitions into
independent problems (frames of a batch), so N GPUs each
filter their own frames with no data-path collective.  One process per GPU
(torchrun); the only collective is the max-over-ranks of the timed region
(plain torch.distributed, NCCL on the GPU box, gloo in the CPU tests).

A single large frame can also be split into row bands: every
output row needs the rho input rows above and below it, so a rank whose band
is already resident exchanges ONE halo of rho rows of f with each neighbour
(point-to-point send / recv, NCCL over NVLink on GPUs) and then filters its
band-plus-halo as an image of its own; theta and sigma are per output pixel
and need no halo, and nothing is exchanged afterwards.  ``band_shard``,
``exchange_halo`` and ``band_problem`` are that host logic.
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


def band_shard(height: int, world: int, rank: int, rho: int = 0) -> tuple[int, int]:
    """Contiguous block of image rows owned by ``rank``: (first, count), counts
    within one row of each other.  With ``rho`` > 0 every band must hold at
    least ``rho`` rows (the halo comes from the adjacent band alone) and the
    band plus its halos at least 2 rho + 1 (the window fits the sub-image)."""
    first, n = frame_shard(height, world, rank)
    if rho > 0 and world > 1:
        smallest = height // world
        if smallest < rho or smallest + rho < 2 * rho + 1:
            raise ValueError(f"bands of {smallest} rows are too thin for rho = {rho} on {world} ranks")
    return first, n


def exchange_halo(band, rho: int, world: int, rank: int):
    """The one exchange step of the band-sharded path: ``band`` is this rank's
    (B, n, W) tensor of image rows (CPU for gloo, CUDA for NCCL).  Sends its
    first / last ``rho`` rows to the rank above / below, receives theirs, and
    returns (band with halos, rows of halo on top).  The first and last rank get
    no halo on the image border: there the filter's own reflection applies."""
    import torch
    import torch.distributed as dist

    if rho == 0 or world == 1:
        return band, 0
    if band.shape[1] < rho:
        raise ValueError("band thinner than rho")
    up = torch.empty_like(band[:, :rho]) if rank > 0 else None
    down = torch.empty_like(band[:, :rho]) if rank < world - 1 else None
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, band[:, :rho].contiguous(), rank - 1))
        ops.append(dist.P2POp(dist.irecv, up, rank - 1))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, band[:, -rho:].contiguous(), rank + 1))
        ops.append(dist.P2POp(dist.irecv, down, rank + 1))
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    parts = ([up] if up is not None else []) + [band] + ([down] if down is not None else [])
    return torch.cat(parts, dim=1), (rho if up is not None else 0)


def band_problem(f_band, theta_band, sigma_band, rho: int, world: int, rank: int):
    """This rank's sub-problem of a row-band split: (f, theta, sigma, top) where f
    carries the exchanged halos, theta / sigma are padded to f's shape (halo rows
    produce outputs that are cropped away: theta = f there, sigma = 1) and
    ``top`` is the first output row to keep; the band's result is
    ``filter(f, theta, sigma)[:, top:top + n]``."""
    import torch

    f, top = exchange_halo(f_band, rho, world, rank)
    n = f_band.shape[1]
    th = f.clone()
    sg = torch.ones_like(f)
    th[:, top:top + n] = theta_band
    sg[:, top:top + n] = sigma_band
    return f, th, sg, top
