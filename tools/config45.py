"""BASELINE configs 4 (AMP, m = 2n) and 5 (spiked GOE power method) on one GPU.
Config 5 is quoted at n = 1e8 over 8 GPUs (n-sharded); one GPU holds n = 1e7.

Env: C4_N, C4_T (0 skips config 4), C5_N, C5_T (0 skips config 5)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat


def config4(n, T):
    m = 2 * n
    g = torch.Generator("cuda").manual_seed(4)
    beta = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) < 0.1) * torch.randn(
        n, device="cuda", generator=g, dtype=torch.float64)
    w = 0.1 * torch.randn(m, device="cuda", generator=g, dtype=torch.float64)
    op = lazymat.GinibreOperator(m, n, m ** -0.5, 4, capacity=T + 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, mse = lazymat.amp_sparse_regression(op, beta, w, T)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    # probe k (1-based over all 2T+1 probes) applies k-1 stored reflectors + the new one
    eu = sum((n if k % 2 == 1 else m) * k for k in range(1, 2 * T + 2))
    return {"n": n, "m": m, "T_amp": T, "probes": 2 * T + 1, "s": dt, "elem_updates_per_s": eu / dt,
            "mse_curve": {str(i): float(mse[i]) for i in list(range(0, T, max(T // 10, 1))) + [T - 1]}}


def config5(n, T):
    g = torch.Generator("cuda").manual_seed(5)
    u = torch.randn(n, device="cuda", generator=g, dtype=torch.float64)
    u /= u.norm()
    x1 = torch.randn(n, device="cuda", generator=g, dtype=torch.float64)
    x1 /= x1.norm()
    op = lazymat.GOEOperator(n, 5, sigma=n ** -0.5, capacity=T)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, ov = lazymat.spiked_power(op, u, x1, T)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    eu = sum(n * k for k in range(1, 2 * T + 1))
    return {"n": n, "T_goe": T, "inner_probes": 2 * T, "s": dt, "elem_updates_per_s": eu / dt,
            "overlap_curve": {str(i): float(ov[i]) for i in list(range(0, T, max(T // 16, 1))) + [T - 1]}}


if __name__ == "__main__":
    res = {}
    n4, T4 = int(os.environ.get("C4_N", 10_000_000)), int(os.environ.get("C4_T", 200))
    n5, T5 = int(os.environ.get("C5_N", 10_000_000)), int(os.environ.get("C5_T", 256))
    if T4:
        res["config4_amp"] = config4(n4, T4)
        torch.cuda.empty_cache()
    if T5:
        res["config5_spiked_goe_1gpu"] = config5(n5, T5)
    print(json.dumps(res, indent=1))
