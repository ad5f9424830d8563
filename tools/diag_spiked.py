import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2101_07464_b200 import lazymat
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
out = {}
for n in [10_000, 100_000, 1_000_000, 10_000_000]:
    T = 120
    g = torch.Generator("cuda").manual_seed(5)
    u = torch.randn(n, device="cuda", generator=g, dtype=torch.float64); u /= u.norm()
    x1 = torch.randn(n, device="cuda", generator=g, dtype=torch.float64); x1 /= x1.norm()
    for ens in ["goe", "haar_sym"]:
        if ens == "goe":
            op = lazymat.GOEOperator(n, 5, sigma=n ** -0.5, capacity=T)
        else:
            continue
        x, ov = lazymat.spiked_power(op, u, x1, T)
        o = ov.cpu().numpy()
        out[f"{ens}_{n}"] = [float(o[i]) for i in (0, 9, 19, 39, 79, 119)]
        # probe norm check on a fresh operator
        op = lazymat.GOEOperator(n, 6, sigma=n ** -0.5, capacity=8)
        ys = []
        xx = x1.clone()
        for t in range(6):
            y = op.probe(xx, "right"); ys.append(float(y.norm())); xx = y / y.norm()
        out[f"{ens}_{n}_norms"] = ys
print(json.dumps(out, indent=1))
