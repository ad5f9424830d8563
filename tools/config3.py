"""BASELINE config 3: B independent Ginibre trials, m = n = 1e5, T = 100,
alternating normalised power iteration, seeds seed + b; fp64 and fp32.
Env: C3_N, C3_B64 / C3_B32 (trials, 0 skips), C3_CONC (operator groups in
flight, comma list), C3_BATCH (trials per batched launch, comma list; 1 = one
graph per trial)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

n, T = int(os.environ.get("C3_N", 100000)), 100
batches = [int(b) for b in os.environ.get("C3_BATCH", "74").split(",")]
res = {}
for dtype, B in (("f64", int(os.environ.get("C3_B64", 1024))), ("f32", int(os.environ.get("C3_B32", 1024)))):
    tdt = torch.float64 if dtype == "f64" else torch.float32
    x1 = torch.randn((B, n), dtype=tdt, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    for conc in [int(c) for c in os.environ.get("C3_CONC", "2").split(",")]:
      for bt in batches:
        if B == 0:
            continue
        # warm-up with the same arguments: allocates the operators, captures the
        # graphs; the timed call reuses them
        _, pool = lazymat.run_trials("ginibre", B, n, T, seed=1, dtype=dtype, concurrency=conc, batch=bt, x1=x1,
                                     return_ops=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = lazymat.run_trials("ginibre", B, n, T, seed=1, dtype=dtype, concurrency=conc, batch=bt, x1=x1,
                                 ops=pool)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        eu = B * n * T * (T + 1) / 2
        key = f"{dtype}_B{B}_conc{conc}" + (f"_batch{bt}" if bt > 1 else "")
        res[key] = {"s": dt, "elem_updates_per_s": eu / dt, "final_norm_mean": float(out.double().norm(dim=1).mean())}
        del pool, out
        torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
