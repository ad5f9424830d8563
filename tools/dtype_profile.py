"""Per-kernel time and achieved bandwidth (algorithmic bytes) of one operator
run in fp64 vs fp32: Haar n = 1e6, T = 100 tanh mix, and Ginibre n = 1e5,
T = 100 alternating normalise (config 3 shape, one trial). Instrumented run."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

res = {}
for ens, n, upd, sides in (("haar", 1_000_000, "tanh_mix", "right"), ("ginibre", 100_000, "normalize", "alternate")):
    for dtype in ("f64", "f32", "f64", "f32"):
        tdt = torch.float64 if dtype == "f64" else torch.float32
        op = (lazymat.HaarOperator(n, seed=1, dtype=dtype, capacity=100) if ens == "haar"
              else lazymat.GinibreOperator(n, n, n ** -0.5, 1, dtype=dtype, capacity=100))
        x1 = torch.randn(n, dtype=tdt, device="cuda")
        x1 /= x1.norm()
        op.run(x1, 100, update=upd, sides=sides)
        op.set_profiling(True)
        op.reset()
        op.run(x1, 100, update=upd, sides=sides)
        st = op.kernel_stats()
        res[f"{ens}_{dtype}"] = {k: (round(v["ms"], 3), round(v["alg_bytes"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] else 0)
                                 for k, v in st.items() if v["ms"] > 0.05}
        print(ens, dtype, res[f"{ens}_{dtype}"], flush=True)
