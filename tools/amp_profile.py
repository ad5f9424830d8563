"""Config-4-shape AMP run (m = 2n) on the device, instrumented: per-kernel-kind
device time and algorithmic-byte rates (CUDA events per launch). For ncu:
run it under `ncu -k regex:k_nt ...` (AP_GRAPH=0 keeps launches visible).

Env: AP_N (default 1e7), AP_T (AMP iterations, default 200), AP_PROF (1: events)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

n = int(float(os.environ.get("AP_N", 1e7)))
T = int(os.environ.get("AP_T", 200))
m = 2 * n
g = torch.Generator("cuda").manual_seed(4)
beta = (torch.rand(n, device="cuda", generator=g, dtype=torch.float64) < 0.1) * torch.randn(
    n, device="cuda", generator=g, dtype=torch.float64)
w = 0.1 * torch.randn(m, device="cuda", generator=g, dtype=torch.float64)
op = lazymat.GinibreOperator(m, n, m ** -0.5, 4, capacity=T + 1)
prof = os.environ.get("AP_PROF", "1") == "1"
op.set_profiling(prof)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
x, mse = lazymat.amp_sparse_regression(op, beta, w, T, use_graph=False)
ev1.record()
torch.cuda.synchronize()
out = {"n": n, "T": T, "ms": ev0.elapsed_time(ev1), "mse_last": float(mse[-1])}
if prof:
    st = op.kernel_stats()
    out["kernels"] = {k: {"launches": v["launches"], "ms": round(v["ms"], 2),
                          "TBps": round(v["alg_bytes"] / (v["ms"] * 1e-3) / 1e12, 2) if v["ms"] else 0}
                      for k, v in st.items()}
print(json.dumps(out, indent=0))
del op  # hd_destroy prints the HD_TRACE=3 breakdown
