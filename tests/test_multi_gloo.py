"""N > 1 host path on CPU (gloo, world size 2): frames shard without overlap
or gaps, the timed region reduces as a max over ranks, and the whole-job rate
counts every rank's pixels over that max (bench.py under torchrun)."""
import os
import socket

import pytest

from paper_1811_02308_b200.shard import band_shard, frame_shard, whole_job_rate


@pytest.mark.parametrize("batch,world", [(32, 1), (32, 2), (32, 8), (5, 2), (3, 4), (0, 2), (7, 7)])
def test_frame_shards_partition_the_batch(batch, world):
    seen = []
    counts = []
    for r in range(world):
        first, n = frame_shard(batch, world, r)
        seen.extend(range(first, first + n))
        counts.append(n)
    assert seen == list(range(batch))
    assert max(counts) - min(counts) <= 1


def test_frame_shard_rejects_bad_rank():
    with pytest.raises(ValueError):
        frame_shard(4, 2, 2)
    with pytest.raises(ValueError):
        frame_shard(4, 0, 0)


def test_whole_job_rate_counts_all_ranks():
    assert whole_job_rate(1_000_000, steps=10, seconds=2.0, world=4) == pytest.approx(20.0)
    assert whole_job_rate([3_000_000, 1_000_000], steps=1, seconds=1.0) == pytest.approx(4.0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1811_02308_b200.shard import frame_shard, max_over_ranks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        first, n = frame_shard(32, world, rank)
        t = max_over_ranks(1.5 + rank)  # each rank's own device time
        q.put((rank, first, n, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    assert [(r, f, n) for r, f, n, _ in res] == [(0, 0, 16), (1, 16, 16)]
    assert all(t == pytest.approx(2.5) for *_, t in res)  # both ranks see the max


def _pipeline_worker(rank, world, port, q):
    """One rank of the sharded path on CPU: its frames of a small batch,
    filtered by the oracle (standing in for the device kernels, which need a
    GPU), gathered back with shard.gather_frames."""
    import numpy as np
    import torch.distributed as dist

    import oracle
    import workloads
    from paper_1811_02308_b200.shard import frame_shard, gather_frames

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = workloads.random_case(5, 20, 23, seed=11, kind="voronoi", rho=2, N=3)
        first, n = frame_shard(5, world, rank)
        sl = slice(first, first + n)
        local = oracle.fast(w.img[sl], w.theta[sl], w.sigma[sl], w.rho, w.N)["g_guard"] if n else np.empty((0, 20, 23))
        full = gather_frames(local, 5, world, rank)
        q.put((rank, n, full))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_pipeline_matches_single_process():
    """World size 2: each rank filters only its frame shard; the gathered
    batch equals the single-process result frame for frame (frames are
    independent problems: no halo, no other collective)."""
    import numpy as np
    import torch.multiprocessing as mp

    import oracle
    import workloads

    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted((q.get(timeout=10) for _ in range(2)), key=lambda t: t[0])
    assert [n for _, n, _ in res] == [3, 2]
    w = workloads.random_case(5, 20, 23, seed=11, kind="voronoi", rho=2, N=3)
    ref = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)["g_guard"]
    for _, _, full in res:
        assert np.array_equal(full, ref)


def test_band_shard_rejects_thin_bands():
    assert band_shard(64, 2, 1, rho=5) == (32, 32)
    with pytest.raises(ValueError):
        band_shard(16, 4, 0, rho=5)


def _band_worker(rank, world, port, q):
    """One rank of the row-band split of a single frame on CPU: its band of f,
    theta, sigma, ONE halo exchange of rho rows of f with each neighbour, the
    band-plus-halo filtered as an image of its own (the oracle standing in for
    the device kernels), cropped to the band."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    import workloads
    from paper_1811_02308_b200.shard import band_problem, band_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = workloads.random_case(2, 41, 29, seed=12, kind="voronoi", rho=4, N=3)
        first, n = band_shard(41, world, rank, rho=w.rho)
        rows = slice(first, first + n)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, rows]))
        f, th, sg, top = band_problem(t(w.img), t(w.theta), t(w.sigma), w.rho, world, rank)
        g = oracle.fast(f.numpy(), th.numpy(), sg.numpy(), w.rho, w.N)["g_guard"][:, top:top + n]
        q.put((rank, first, n, tuple(f.shape), g))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_band_split_matches_single_process(world):
    """A single frame split into row bands over 2 and 3 ranks: after the one
    halo exchange every rank's cropped result equals the corresponding rows of
    the single-process result (interior ranks carry a halo on both sides, the
    border ranks rely on the filter's own reflection)."""
    import numpy as np
    import torch.multiprocessing as mp

    import oracle
    import workloads

    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    res = sorted((q.get(timeout=10) for _ in range(world)), key=lambda t: t[0])
    w = workloads.random_case(2, 41, 29, seed=12, kind="voronoi", rho=4, N=3)
    ref = oracle.fast(w.img, w.theta, w.sigma, w.rho, w.N)["g_guard"]
    rows = 0
    for rank, first, n, shape, g in res:
        halos = (rank > 0) + (rank < world - 1)
        assert shape == (2, n + halos * w.rho, 29)
        assert np.array_equal(g, ref[:, first:first + n])
        rows += n
    assert rows == 41
