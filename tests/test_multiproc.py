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
        val = bench.whole_job_value(world, bench.eu_haar(1000, 10), 3, mx)
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


# ------------------------------------------------ row-sharded operators (e1)
def _shard_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2101_07464_b200 import lazymat as lm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plans = {}
        for N, head in [(10 ** 8, 768), (2 * 10 ** 7, 512), (3001, 256), (1800, 256)]:
            got = [None] * world
            dist.all_gather_object(got, lm.shard_plan(N, world, rank, head))
            plans[N] = (head, got)
        ids = [None] * world
        dist.all_gather_object(ids, lm.share_nccl_id())
        q.put((rank, plans, ids))
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_plan_and_nccl_id():
    # host logic of the n-sharded operator: every rank derives the same
    # tile-aligned row slabs (disjoint, covering [0, N), shard 0 holding the
    # head rows) and the same NCCL id from rank 0
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, plans0, ids0), (_, plans1, ids1) = res
    assert plans0 == plans1
    for N, (head, ranges) in plans0.items():
        assert ranges[0][0] == 0 and ranges[-1][1] == N and ranges[0][1] >= head
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert b == c and a < b and b % 256 == 0
    assert ids0[0] == ids0[1] == ids1[0] and len(ids0[0]) == 128


def test_bench_self_spawns_ranks_and_plans_config5_slabs():
    # `python bench.py --gpus 2` launches its own 2 ranks (torch.distributed.run);
    # the CPU self-test runs the multi-rank plumbing over gloo: each rank's row
    # slab of config 5's n (hd_shard_plan), max-over-ranks timing, whole-job value
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dist-selftest",
                          "--n5", "1000000", "--T5", "16"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["selftest"] == "ok" and line["world"] == 2
    assert line["ms"] == 11.0  # the slowest rank's time
    (lo0, hi0), (lo1, hi1) = line["slabs"]
    assert lo0 == 0 and hi0 == lo1 and hi1 == 2_000_000 and hi0 % 256 == 0
