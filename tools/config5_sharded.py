"""BASELINE config 5 — spiked GOE power method x <- (Q x + theta <u,x> u)/||.||,
inner sigma = 1/sqrt(n), theta = 2, T = 256 GOE steps — with the operator
row-sharded across the ranks of a torchrun job (one GPU each): every rank
owns a row slab (lazymat.shard_plan) and runs the whole dynamics device-
resident (lazymat.spiked_power -> hd_run_spiked): the probes' partial dots and
the map's sums (<u, x>, ||g||^2) travel in the operator's NCCL exchange
(lazymat.nccl_exchange), so the loop has no torch.distributed calls and no
per-probe host synchronisation. Quoted at n = 1e8 on 8 GPUs; C5_N sets n
(default 1.25e7 per rank, i.e. weak scaling to 1e8 at 8 ranks).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/config5_sharded.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2101_07464_b200 import lazymat


def main():
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    n = int(float(os.environ.get("C5_N", 12_500_000 * world)))
    T = int(os.environ.get("C5_T", 256))
    theta = 2.0
    ex = lazymat.nccl_exchange()
    op = lazymat.GOEOperator(n, 5, sigma=n ** -0.5, capacity=T, shard=(rank, world), exchange=ex)
    lo, hi = op.shard_range()
    # the same u, x_1 on every rank (seeded device generator), sliced to the slab
    g = torch.Generator("cuda").manual_seed(5)
    u = torch.randn(n, device="cuda", generator=g, dtype=torch.float64)
    x = torch.randn(n, device="cuda", generator=g, dtype=torch.float64)
    u, x = (u / u.norm())[lo:hi].clone(), (x / x.norm())[lo:hi].clone()
    torch.cuda.empty_cache()

    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    x, ov = lazymat.spiked_power(op, u, x, T, theta=theta)
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    eu = n * (2 * T) * (2 * T + 1) / 2  # inner probe k touches n * k elements
    if rank == 0:
        print(json.dumps({"workload": "config5 spiked GOE, row-sharded", "n": n, "ranks": world, "T_goe": T,
                          "s": ms.item() / 1e3, "wall_s": wall, "elem_updates_per_s": eu / (ms.item() / 1e3),
                          "overlap_curve": {str(i): float(ov[i]) for i in list(range(0, T, 32)) + [T - 1]}}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
