"""Per-probe latency floor: small-n runs where launch/latency dominates."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

out = {}
for ens, n, T in (("haar", 4096, 100), ("haar", 100000, 100), ("ginibre", 4096, 50)):
    op = (lazymat.HaarOperator(n, seed=1, capacity=T) if ens == "haar"
          else lazymat.GinibreOperator(n, n, sigma=n ** -0.5, seed=1, capacity=T))
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    upd, sides = ("tanh_mix", "right") if ens == "haar" else ("normalize", "alternate")
    for g in (False, True):
        for _ in range(3):
            op.reset(); op.run(x, T, update=upd, sides=sides, use_graph=g)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            op.reset(); op.run(x, T, update=upd, sides=sides, use_graph=g)
        b.record(); torch.cuda.synchronize()
        out[f"{ens}_n{n}_T{T}_graph{int(g)}_us_per_probe"] = a.elapsed_time(b) / 5 / T * 1e3
print(json.dumps(out))
