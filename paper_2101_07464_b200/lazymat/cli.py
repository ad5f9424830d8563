"""`lazymat bench` on the device path: the reference CLI's wall-clock scaling
subcommand (tools/lazymat_cli.cpp:384-494, src/bench.cpp:17-150) with the same
flags, defaults, CSV schema (`backend,n,T,median_ms`), manifest (config
round-trip, log-log slopes, `deterministic: false`), `--from-manifest` replay and
exit codes (0 ok, 2 usage, 4 resource cap; lazymat_cli.cpp:32-35).

The timed workload is the reference's (bench.cpp:35-54): a square Ginibre
operator with sigma = 1/sqrt(n) built from a seed, T probes alternating right /
left from x_1 = 1/sqrt(n) (1, ..., 1), each output normalised; the clock covers
operator construction and the run. `hd` is the device operator (one device-
resident run, device Philox draws); `direct` materialises the dense Ginibre
matrix in HBM (the reference's DenseOperator over sample_dense_ginibre, capped
by LAZYMAT_ORACLE_DIM_CAP / --dim-cap) and applies it with dense GEMVs.

    python -m paper_2101_07464_b200.lazymat.cli --out DIR bench [--backend hd|direct|both] ...
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

VERSION = "0.1.0"
EXIT_OK, EXIT_USAGE, EXIT_VERIFY_FAILED, EXIT_RESOURCE_CAP = 0, 2, 3, 4

BENCH_DEFAULTS = {"backend": "hd", "nmin": 0, "nmax": 0, "T": 50, "reps": 3, "fix_n": False, "fixed_n": 16384,
                  "sweep_T": [10, 20, 40, 80], "seed": 1, "dim_cap": 0}


class UsageError(ValueError):
    pass


def fmt_double(v: float) -> str:
    return "%.17g" % v  # lazymat_cli.cpp:37-41


def iso_now() -> str:
    return time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())


def warn_if_loaded() -> None:  # lazymat_cli.cpp:421-431
    try:
        load1 = float(open("/proc/loadavg").read().split()[0])
    except Exception:
        return
    cores = max(1, os.cpu_count() or 1)
    if load1 > 0.5 * cores:
        print(f"warning: system load {load1:g} on {cores} cores; timings may be noisy", file=sys.stderr)


def power_grid(lo: int, hi: int):  # lazymat_cli.cpp:433-438
    if not (lo >= 1 and lo <= hi):
        raise UsageError("bench: need 1 <= nmin <= nmax")
    grid, n = [], lo
    while n <= hi:
        grid.append(n)
        n *= 2
    return grid


def median_of(xs):  # bench.cpp:56-62
    if not xs:
        raise UsageError("median_of: empty sample")
    xs = sorted(xs)
    k = len(xs) // 2
    return xs[k] if len(xs) % 2 == 1 else 0.5 * (xs[k - 1] + xs[k])


def fit_loglog(x, y) -> float:  # bench.cpp:95-122
    if len(x) != len(y) or len(x) < 2:
        raise UsageError("fit_loglog: need matched samples with at least two points")
    if any(v <= 0 for v in list(x) + list(y)):
        raise UsageError("fit_loglog: inputs must be positive")
    lx, ly = [math.log(v) for v in x], [math.log(v) for v in y]
    mx, my = sum(lx) / len(lx), sum(ly) / len(ly)
    sxy = sum((a - mx) * (b - my) for a, b in zip(lx, ly))
    sxx = sum((a - mx) ** 2 for a in lx)
    if not sxx > 0:
        raise UsageError("fit_loglog: abscissae must not be constant")
    return sxy / sxx


def time_workload_ms(backend: str, n: int, T: int, seed: int, dim_cap: int) -> float:
    """bench.cpp:35-54 on the device: construction + T alternating normalised probes."""
    import torch

    from . import GinibreOperator, RandomSource
    from .experiments import _dense_ginibre

    if not (n >= 1 and T >= 1):
        raise UsageError("time_workload_ms: n and T must be positive")
    if T > n:
        raise UsageError("time_workload_ms: probe budget needs T <= n")
    sigma = 1.0 / math.sqrt(n)
    x1 = torch.full((n,), 1.0 / math.sqrt(n), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if backend == "hd":
        op = GinibreOperator(n, n, sigma, seed, capacity=T)
        op.run(x1, T, update="normalize", sides="alternate", use_graph=False)
    else:
        old = os.environ.get("LAZYMAT_ORACLE_DIM_CAP")
        if dim_cap > 0:
            os.environ["LAZYMAT_ORACLE_DIM_CAP"] = str(dim_cap)
        try:
            a = _dense_ginibre(n, n, sigma, RandomSource(seed, 0))
        finally:
            if dim_cap > 0:
                if old is None:
                    os.environ.pop("LAZYMAT_ORACLE_DIM_CAP", None)
                else:
                    os.environ["LAZYMAT_ORACLE_DIM_CAP"] = old
        x = x1
        for t in range(1, T + 1):
            y = a @ x if t % 2 == 1 else a.t() @ x
            nrm = torch.linalg.vector_norm(y)
            x = y * torch.where(nrm > 0, 1.0 / nrm, torch.ones_like(nrm))
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)


def measure(backend, n, T, cfg, salt):  # bench.cpp:66-78
    from . import derive_seed

    if cfg["reps"] < 1:
        raise UsageError("bench: reps must be positive")
    times = [time_workload_ms(backend, n, T, derive_seed(cfg["seed"], salt * 64 + r), cfg["dim_cap"])
             for r in range(cfg["reps"])]
    return {"backend": backend, "n": n, "T": T, "median_ms": median_of(times)}


def run_bench(cfg: dict, out_dir: str) -> int:  # lazymat_cli.cpp:440-494
    warn_if_loaded()
    backends = ["hd", "direct"] if cfg["backend"] == "both" else [cfg["backend"]]
    csv = "backend,n,T,median_ms\n"
    slopes, summary = [], ""
    for b in backends:
        if cfg["fix_n"]:
            pts = [measure(b, cfg["fixed_n"], T, cfg, 1000 + i) for i, T in enumerate(cfg["sweep_T"])]
            slope = fit_loglog([p["T"] for p in pts], [p["median_ms"] for p in pts])
            axis = "T"
        else:
            lo = cfg["nmin"] if cfg["nmin"] > 0 else (4096 if b == "hd" else 512)
            hi = cfg["nmax"] if cfg["nmax"] > 0 else (131072 if b == "hd" else 4096)
            pts = [measure(b, n, cfg["T"], cfg, i + 1) for i, n in enumerate(power_grid(lo, hi))]
            slope = fit_loglog([p["n"] for p in pts], [p["median_ms"] for p in pts])
            axis = "n"
        for p in pts:
            csv += f"{p['backend']},{p['n']},{p['T']},{fmt_double(p['median_ms'])}\n"
        summary += "slope(backend=%s, axis=%s) = %.3f\n" % (b, axis, slope)
        slopes.append({"backend": b, "axis": axis, "slope": slope})
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, "bench.csv")
    with open(path, "w") as f:
        f.write(csv)
    manifest = {"subcommand": "bench", "config": cfg, "outputs": ["bench.csv"], "slopes": slopes,
                "deterministic": False,  # configuration round-trips exactly; measured times never do
                "tool": "lazymat", "version": VERSION, "generated_at": iso_now()}
    with open(os.path.join(out_dir, "bench_manifest.json"), "w") as f:
        f.write(json.dumps(manifest, indent=2) + "\n")
    print(f"wrote {path}\n{summary}", end="")
    return EXIT_OK


def bench_config_from_json(j: dict) -> dict:  # lazymat_cli.cpp:407-419 (every key required)
    cfg = {}
    for k in BENCH_DEFAULTS:
        if k not in j:
            raise UsageError(f"manifest config lacks '{k}'")
        cfg[k] = j[k]
    return cfg


def run_from_manifest(path: str, out_dir: str) -> int:  # lazymat_cli.cpp:498-514
    try:
        manifest = json.load(open(path))
    except OSError:
        raise UsageError(f"cannot read manifest {path}")
    sub = manifest.get("subcommand")
    if sub == "bench":
        return run_bench(bench_config_from_json(manifest["config"]), out_dir)
    raise UsageError(f"manifest names unknown subcommand: {sub}")


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 parse errors exit with the usage code
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        sys.exit(EXIT_USAGE)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="lazymat", description="matrix-free random-ensemble simulation toolkit (B200 device path)")
    ap.add_argument("--version", action="version", version=VERSION)
    ap.add_argument("--out", default=".", help="output directory")
    ap.add_argument("--from-manifest", default="", help="re-run the configuration stored in a manifest")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    b = sub.add_parser("bench", help="wall-clock scaling; single-threaded")
    b.add_argument("--backend", default="hd", choices=["hd", "direct", "both"], help="hd, direct, or both")
    b.add_argument("--nmin", type=int, default=0, help="smallest n (0 = backend default)")
    b.add_argument("--nmax", type=int, default=0, help="largest n (0 = backend default)")
    b.add_argument("--T", "-T", type=int, default=50, help="probes per run")
    b.add_argument("--reps", type=int, default=3, help="repetitions per point")
    b.add_argument("--fix-n", action="store_true", help="sweep T at fixed n instead of sweeping n")
    b.add_argument("--fixed-n", type=int, default=16384, help="n used with --fix-n")
    b.add_argument("--sweep-T", type=int, nargs="+", default=[10, 20, 40, 80], help="T grid used with --fix-n")
    b.add_argument("--seed", type=int, default=1, help="base seed")
    b.add_argument("--dim-cap", type=int, default=0, help="dense-oracle dimension cap override (0 = default)")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    from .. import _native as N

    try:
        os.makedirs(args.out, exist_ok=True)
        if args.from_manifest:
            if args.cmd:
                print("error: --from-manifest replaces the subcommand", file=sys.stderr)
                return EXIT_USAGE
            return run_from_manifest(args.from_manifest, args.out)
        if args.cmd == "bench":
            cfg = {"backend": args.backend, "nmin": args.nmin, "nmax": args.nmax, "T": args.T, "reps": args.reps,
                   "fix_n": bool(args.fix_n), "fixed_n": args.fixed_n, "sweep_T": list(args.sweep_T),
                   "seed": args.seed, "dim_cap": args.dim_cap}
            return run_bench(cfg, args.out)
        ap.print_help(sys.stderr)
        return EXIT_USAGE
    except N.ResourceCapExceeded as e:
        print(f"resource cap: {e}", file=sys.stderr)
        return EXIT_RESOURCE_CAP
    except N.BudgetExhausted as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (UsageError, ValueError) as e:
        print(f"usage error: {e}", file=sys.stderr)
        print("run with --help for flag documentation", file=sys.stderr)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
