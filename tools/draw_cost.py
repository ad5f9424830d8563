import os, sys, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2101_07464_b200 import lazymat
n, T = 1_000_000, 100
dtype = os.environ.get("DTYPE", "f64")
tdt = torch.float64 if dtype == "f64" else torch.float32
res = {}
for mode in ["philox", "injected", "philox"]:
    op = lazymat.HaarOperator(n, seed=1, draws=mode, capacity=T, dtype=dtype)
    if mode == "injected":
        g = torch.Generator().manual_seed(1)
        op.push_draws(torch.randn(n * (T + 1), dtype=torch.float64, generator=g).numpy())
    op.set_profiling(True)
    x1 = torch.randn(n, dtype=tdt, device="cuda"); x1 /= x1.norm()
    op.run(x1, T, update="tanh_mix", sides="right")
    st = op.kernel_stats()
    res[mode] = {k: round(v["ms"], 3) for k, v in st.items()}
    print(mode, res[mode], flush=True)
