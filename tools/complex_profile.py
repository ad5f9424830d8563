import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, json
from paper_2101_07464_b200 import lazymat
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
op = lazymat.HaarOperator(n, seed=1, dtype="c128", capacity=T)
op.set_profiling(True)
x = torch.randn(n, dtype=torch.complex128, device="cuda"); x /= x.norm()
for t in range(T):
    y = op.probe(x, "right"); x = y / y.norm()
st = op.kernel_stats()
print(json.dumps({k: {"launches": v["launches"], "ms": round(v["ms"], 3), "GB": round(v["alg_bytes"] / 1e9, 2),
                      "GBps": round(v["alg_bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else 0} for k, v in st.items()}, indent=0))
