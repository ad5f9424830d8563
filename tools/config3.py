"""BASELINE config 3: B independent Ginibre trials, m = n = 1e5, T = 100,
alternating normalised power iteration, seeds seed + b; fp64 and fp32."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

n, T = int(os.environ.get("C3_N", 100000)), 100
res = {}
for dtype, B in (("f64", int(os.environ.get("C3_B64", 1024))), ("f32", int(os.environ.get("C3_B32", 1024)))):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    x1 = torch.randn((B, n), dtype=tdt, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    for conc in [int(c) for c in os.environ.get("C3_CONC", "16").split(",")]:
        lazymat.run_trials("ginibre", min(B, 2 * conc), n, T, seed=1, dtype=dtype, concurrency=conc,
                           x1=x1[: min(B, 2 * conc)])  # warm: capture graphs
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = lazymat.run_trials("ginibre", B, n, T, seed=1, dtype=dtype, concurrency=conc, x1=x1)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        eu = B * n * T * (T + 1) / 2
        res[f"{dtype}_B{B}_conc{conc}"] = {"s": dt, "elem_updates_per_s": eu / dt,
                                           "final_norm_mean": float(out.double().norm(dim=1).mean())}
print(json.dumps(res, indent=1))
