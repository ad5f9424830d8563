#!/usr/bin/env python
"""Benchmark of the HD hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the headline single-GPU config):
  Haar-orthogonal HD operator, n = 1e6, T = 100 probes (all Q x), fp64,
  x_1 = g/||g|| (seeded), x_0 = 0, dynamics x_{t+1} = tanh(2 Q x_t) + 0.1 x_{t-1}.
A step = one full T-probe HD run on a freshly reset operator (device Philox
draws). Metric: HD element-updates/s = sum_t n*t per run / time.

--gpus N > 1 runs one independent trial per rank (trial sharding, no
data-path collective, scaling "weak"); time = max over ranks (CUDA events).
--impl reference times the reference's CPU path (the oracle restatement in
oracle/, since the reference itself cannot be built here — DESIGN.md) with
all host threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 1_000_000
T_DEFAULT = 100
METRIC = "HD element-updates/s (n*t per probe, summed over the run)"
UNIT = "element-updates/s"


def elem_updates(n: int, T: int) -> float:
    return float(n) * T * (T + 1) / 2.0


def alg_bytes_haar(n: int, T: int, s: int = 8) -> float:
    """SURVEY §8d Haar probe: s*n*(3t+2) summed over t = 1..T."""
    return float(s) * n * (3.0 * T * (T + 1) / 2.0 + 2.0 * T)


def alg_bytes_haar_2p(n: int, T: int, s: int = 8) -> float:
    """Two-pass Haar run: s*n*(2t+4) summed over t = 1..T
    (the other panel's t and the fold panel's t - 1 columns read once, the new
    fold column, x_t, x_{t+1}, x_{t-1} and the next mix column)."""
    return float(s) * n * (2.0 * T * (T + 1) / 2.0 + 4.0 * T)


def rank_seed(base: int, rank: int) -> int:
    """One independent trial per rank (trial sharding)."""
    return base + 1000 * rank


def shard_trials(total: int, world: int, rank: int):
    """Contiguous trial range of `rank` (batched-trial configs)."""
    return (total * rank // world, total * (rank + 1) // world)


def max_over_ranks(x: float, dist, device) -> float:
    import torch

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(world: int, n: int, T: int, steps: int, ms: float) -> float:
    """Aggregate element-updates/s over all ranks, timed by the slowest rank."""
    return world * elem_updates(n, T) * steps / (ms / 1e3)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.out = None

    def __enter__(self):
        try:
            self.out = open(os.devnull if False else "/tmp/hd_clocks.csv", "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.out:
            self.out.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open("/tmp/hd_clocks.csv").read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 4 + k and "Active" in r[4 + k] and "Not" not in r[4 + k]:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(n: int, T_sample: int, seed: int):
    """The reference hot path restated (oracle/, -O3 -mavx2 -mfma) single-threaded
    like run_dynamics; one Haar trial of T_sample probes (bounded sample)."""
    from oracle import oracle as orc

    orc.build()
    secs, _ = orc.bench_workload("haar", n, n, 1.0, "tanh_mix", "right", T_sample, seed, 1, 1)
    return {"value": elem_updates(n, T_sample) / secs, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"1 trial, Haar n={n}, T={T_sample} probes (tanh mix), {secs:.2f} s wall incl. construction; "
                      f"CPU {cpu_model()}"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.build()
    threads = max(1, min(os.cpu_count() or 1, args.ref_threads))
    n, T_s = args.n, args.ref_T
    trials = threads
    times = []
    for i in range(args.warmup + args.steps):
        secs, _ = orc.bench_workload("haar", n, n, 1.0, "tanh_mix", "right", T_s, args.seed + i, trials, threads)
        if i >= args.warmup:
            times.append(secs)
    per = elem_updates(n, T_s) * trials
    tot = sum(times)
    value = per * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{trials} concurrent Haar trials (one per thread), n={n}, T={T_s} probes each, "
                                   f"tanh mix; CPU {cpu_model()}, nproc={os.cpu_count()}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baselines_all(args):
    """The reference CPU path (oracle port, -O3 -mavx2 -mfma) timed on this
    host for the other BASELINE configs, on bounded samples; where the full
    config exceeds a few seconds (or host RAM) the sample is smaller and the
    full-config time is extrapolated from the measured element-update rate
    (the reference's n-slope is ~1, acceptance.cpp:206-218)."""
    import time

    from oracle import oracle as orc

    orc.build()
    threads = max(1, min(os.cpu_count() or 1, args.ref_threads))
    out = []

    def emit(workload, sample, eu, secs, threads_used, full_eu):
        rate = eu / secs
        out.append({"impl": "reference", "workload": workload, "sample": sample, "cpu_elem_updates_per_s": rate,
                    "threads": threads_used, "sample_s": secs, "full_config_elem_updates": full_eu,
                    "extrapolated_full_config_s": full_eu / rate, "cpu": cpu_model(), "nproc": os.cpu_count()})

    def gin_eu(n, T):  # square Ginibre, alternating: probe k touches n k
        return n * T * (T + 1) / 2

    # config 1: full size, one trial, one thread (run_dynamics is serial)
    secs, _ = orc.bench_workload("ginibre", 4096, 4096, 4096 ** -0.5, "normalize", "alternate", 50, 1, 1, 1)
    emit("config1_ginibre_4096_T50", "full config, 1 trial, 1 thread", gin_eu(4096, 50), secs, 1, gin_eu(4096, 50))
    # config 3: `threads` trials of the 1024 (one per thread, parallel_for)
    n, T = 100_000, 100
    secs, _ = orc.bench_workload("ginibre", n, n, n ** -0.5, "normalize", "alternate", T, 1, threads, threads)
    emit("config3_ginibre_1e5_T100_B1024", f"{threads} of the 1024 trials, one per thread", gin_eu(n, T) * threads,
         secs, threads, gin_eu(n, T) * 1024)
    # config 4: AMP at n = 1e5 (m = 2n), 50 AMP iterations (101 probes), 1 thread
    n, T = 100_000, 50
    m = 2 * n
    rs = orc.RandomSource(4, 1)
    beta = np.array([(rs.uniform() < 0.1) * rs.normal() for _ in range(n)])
    w = 0.1 * rs.normal_vector(m)
    op = orc.Operator("ginibre", m=m, n=n, sigma=m ** -0.5, seed=4)
    t0 = time.perf_counter()
    op.amp(beta, w, T)
    secs = time.perf_counter() - t0
    eu = lambda nn, TT: sum((nn if k % 2 == 1 else 2 * nn) * k for k in range(1, 2 * TT + 2))  # noqa: E731
    emit("config4_amp_n1e7_T200", "n = 1e5 (m = 2e5), 50 AMP iterations, 1 thread", eu(n, T), secs, 1,
         eu(10_000_000, 200))
    # config 5: spiked GOE at n = 1e5, 64 steps (128 inner probes), 1 thread
    n, T = 100_000, 64
    u = orc.RandomSource(5, 1).normal_vector(n)
    u /= np.linalg.norm(u)
    x1 = orc.RandomSource(5, 2).normal_vector(n)
    x1 /= np.linalg.norm(x1)
    op = orc.Operator("goe", n=n, sigma=n ** -0.5, seed=5)
    t0 = time.perf_counter()
    op.spiked_power(u, x1, T)
    secs = time.perf_counter() - t0
    emit("config5_spiked_goe_n1e8_T256", "n = 1e5, 64 GOE steps (128 inner probes), 1 thread", gin_eu(n, 2 * T),
         secs, 1, gin_eu(100_000_000, 512))
    for line in out:
        print(json.dumps(line), flush=True)


def workload_config(args):
    return {"workload": f"config2_haar_n{args.n}_T{args.T}_tanh_mix", "ensemble": "haar", "n": args.n,
            "T": args.T, "dynamics": "x_{t+1}=tanh(2Qx_t)+0.1x_{t-1}", "draws": "device philox4x32-10",
            "trials_per_gpu": 1, "l2": "inputs larger than L2 (2 panels x n x T x 8 B = "
                                        f"{2 * args.n * args.T * 8 / 1e9:.2f} GB > 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)  # ~0.8 s timed: several nvidia-smi clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=N_DEFAULT)
    ap.add_argument("--T", type=int, default=T_DEFAULT)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-T", type=int, default=60, help="probes in the bounded cpu_baseline sample")
    ap.add_argument("--ref-T", type=int, default=30, help="probes per trial in the reference arm sample")
    ap.add_argument("--ref-threads", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-baselines", action="store_true",
                    help="time the reference CPU path (oracle) on configs 1, 3, 4, 5 and exit")
    args = ap.parse_args()

    if args.cpu_baselines:
        import numpy as np  # noqa: F401  (used by cpu_baselines_all)

        globals()["np"] = np
        cpu_baselines_all(args)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import __graft_entry__ as ge

    if rank == 0:
        ge.build()
    if world > 1:
        dist.barrier()
    from paper_2101_07464_b200 import lazymat

    n, T = args.n, args.T
    seed = rank_seed(args.seed, rank)
    op = lazymat.HaarOperator(n, seed=seed, capacity=T, device=local)
    gen = torch.Generator(device=dev).manual_seed(seed)
    x1 = torch.randn(n, dtype=torch.float64, device=dev, generator=gen)
    x1 /= x1.norm()
    x0 = torch.zeros(n, dtype=torch.float64, device=dev)
    use_graph = not args.no_graph

    def step_device():
        # fresh operator, same seed: reseed resets the host counters without a
        # host sync (the captured graph resets the device state itself), so the
        # timed region holds back-to-back graph replays
        op.reseed(seed)
        return op.run(x1, T, update="tanh_mix", sides="right", x0=x0, use_graph=use_graph)

    for _ in range(max(args.warmup, 3)):
        step_device()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = op.launch_count()
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            out = step_device()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = (op.launch_count() - l0) // args.steps
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        ms = max_over_ranks(ms, dist, dev)
        dist.barrier()
    ms_step = ms / args.steps
    value = whole_job_value(world, n, T, args.steps, ms)
    final_norm = float(out.norm())

    # e2e through the public API with host buffers in pinned memory (H2D x_1;
    # x_0 = 0 is the library's default history; D2H x_{T+1}), every step
    # inside the timed region, each on a fresh operator (reseed)
    x1p = x1.cpu().pin_memory()
    outp = torch.empty(n, dtype=torch.float64).pin_memory()
    x1h, outh = x1p.numpy(), outp.numpy()
    op.reseed(seed)
    op.run(x1h, T, update="tanh_mix", sides="right", use_graph=use_graph, out=outh)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.reseed(seed)
        op.run(x1h, T, update="tanh_mix", sides="right", use_graph=use_graph, out=outh)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        e2e_s = max_over_ranks(e2e_s, dist, dev)
    e2e_val = whole_job_value(world, n, T, args.steps, e2e_s * 1e3)
    assert np.isfinite(outh).all()

    # roofline: instrumented pass (CUDA events around every launch on the op's stream)
    op.reset()
    op.set_profiling(True)
    op.reset_stats()
    op.run(x1, T, update="tanh_mix", sides="right", x0=x0, use_graph=False)
    stats = op.kernel_stats()
    op.set_profiling(False)
    peak, peak_kind = load_peaks()
    dom = max((k for k in stats if stats[k]["alg_bytes"] > 0), key=lambda k: stats[k]["ms"])
    d = stats[dom]
    achieved = (d["alg_bytes"] / d["launches"]) / (d["ms"] / d["launches"] / 1e3) / 1e9
    tot_ms = sum(v["ms"] for v in stats.values())
    tot_bytes = sum(v["alg_bytes"] for v in stats.values())
    # DRAM bytes per launch of the dominant kernel: the committed ncu capture's
    # DRAM/algorithmic ratio (probe t = 91) applied to this run's per-launch bytes
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tr = json.load(open(tp)).get(dom)
            if tr:
                traffic = tr["ratio"] * d["alg_bytes"] / d["launches"]
        except Exception:
            traffic = None

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (device Philox draws, seeded x_1)",
            "config": workload_config(args),
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                         "peak_source": peak_kind,
                         "kernel_share_of_step": d["ms"] / tot_ms if tot_ms else None,
                         "method": "per-launch CUDA events on the operator's stream (the stream the kernels "
                                   "run on) in an instrumented, non-graph run of the same workload right after "
                                   "the timed region (events cannot sit between kernels of a graph replay); "
                                   "achieved = algorithmic bytes per launch / mean launch duration",
                         "step_alg_GBps": tot_bytes / (tot_ms / 1e3) / 1e9 if tot_ms else None,
                         "survey_formula_GBps": alg_bytes_haar(n, T) / (ms_step / 1e3) / 1e9,
                         "two_pass_formula_GBps": alg_bytes_haar_2p(n, T) / (ms_step / 1e3) / 1e9,
                         "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 4),
                                         "alg_GB": round(v["alg_bytes"] / 1e9, 4)} for k, v in stats.items()}},
            "clocks": clocks,
            "final_norm": final_norm,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(n, min(args.cpu_T, T), args.seed)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
