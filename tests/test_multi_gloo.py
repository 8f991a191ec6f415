"""N > 1 host path on CPU (gloo, world size 2): frames shard without overlap
or gaps, the timed region reduces as a max over ranks, and the whole-job rate
counts every rank's pixels over that max (bench.py under torchrun)."""
import os
import socket

import pytest

from paper_1811_02308_b200.shard import frame_shard, whole_job_rate


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
