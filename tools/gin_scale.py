"""Ginibre / GOE throughput at scale (Philox draws, normalise dynamics)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

def run(make, n, T, sides, reps=3):
    op = make()
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        op.reset(); op.run(x, T, update="normalize", sides=sides, use_graph=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        op.reset(); op.run(x, T, update="normalize", sides=sides, use_graph=True)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    op.reset(); op.set_profiling(True); op.reset_stats()
    op.run(x, T, update="normalize", sides=sides)
    st = {k: round(v["ms"], 3) for k, v in op.kernel_stats().items()}
    return ms, st

out = {}
n, T = 1_000_000, 100
ms, st = run(lambda: lazymat.GinibreOperator(n, n, sigma=n ** -0.5, seed=1, capacity=T), n, T, "alternate")
out["ginibre_n1e6_T100_alt"] = {"ms": ms, "elem_updates_per_s": n * T * (T + 1) / 2 / (ms / 1e3), "kernels": st}
n, T = 4096, 50
ms, st = run(lambda: lazymat.GinibreOperator(n, n, sigma=n ** -0.5, seed=1, capacity=T), n, T, "alternate", reps=10)
out["ginibre_n4096_T50_alt(config1)"] = {"ms": ms, "elem_updates_per_s": n * T * (T + 1) / 2 / (ms / 1e3), "kernels": st}
n, T = 1_000_000, 50
ms, st = run(lambda: lazymat.GOEOperator(n, seed=1, sigma=n ** -0.5, capacity=T), n, T, "right")
out["goe_n1e6_T50"] = {"ms": ms, "elem_updates_per_s": n * (2 * T) * (2 * T + 1) / 2 / (ms / 1e3), "kernels": st}
print(json.dumps(out, indent=1))
