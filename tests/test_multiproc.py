"""World-size-2 (gloo, CPU) checks of the multi-rank host logic of bench.py:
one independent trial per rank (trial sharding, no data-path collective),
the max-over-ranks timing and the whole-job aggregate."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import bench

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms = 10.0 + 5.0 * rank  # rank 1 is the slow one
        mx = bench.max_over_ranks(ms, dist, torch.device("cpu"))
        seeds = [None] * world
        dist.all_gather_object(seeds, bench.rank_seed(1, rank))
        shards = [None] * world
        dist.all_gather_object(shards, bench.shard_trials(1024, world, rank))
        val = bench.whole_job_value(world, 1000, 10, 3, mx)
        q.put((rank, mx, seeds, shards, val))
    finally:
        dist.destroy_process_group()


def test_two_rank_trial_sharding_and_timing():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, seeds, shards, val in res:
        assert mx == 15.0  # slowest rank defines the job time
        assert len(set(seeds)) == world  # independent trials
        assert shards == [(0, 512), (512, 1024)]
        assert val == pytest.approx(2 * 1000 * 55 * 3 / 0.015)
