"""Per-kernel device time / algorithmic bytes of a Ginibre run (config 4 shape:
m = 2n, alternating probes, normalise), instrumented (events per launch)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
n = int(float(os.environ.get("GP_N", 1e7)))
m, T = 2 * n, int(os.environ.get("GP_T", 60))
op = lazymat.GinibreOperator(m, n, m ** -0.5, 4, capacity=T)
op.set_profiling(True)
x1 = torch.randn(n, dtype=torch.float64, device="cuda")
op.run(x1, T, update="normalize", sides="alternate")
st = op.kernel_stats()
print(json.dumps({k: {"launches": v["launches"], "ms": round(v["ms"], 2),
                      "TBps": round(v["alg_bytes"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] else 0}
                  for k, v in st.items()}, indent=0))
