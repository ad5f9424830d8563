"""Throughput of the complex-field operators (f2): probes of a Haar (n = 1e6)
and a Ginibre (m = n = 1e5) operator over complex<double>, Philox draws."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

res = {}
TH = int(sys.argv[1]) if len(sys.argv) > 1 else 30
NG = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000
TG = int(sys.argv[3]) if len(sys.argv) > 3 else 40
for ens, n, T in [("haar", 1_000_000, TH), ("ginibre", NG, TG)]:
    op = (lazymat.HaarOperator(n, seed=1, dtype="c128", capacity=T) if ens == "haar"
          else lazymat.GinibreOperator(n, n, n ** -0.5, 1, dtype="c128", capacity=T))
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    x /= x.norm()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(T):
        y = op.probe(x, "right" if (ens == "haar" or t % 2 == 0) else "left")
        x = y / y.norm()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    eu = n * T * (T + 1) / 2
    res[ens] = {"n": n, "probes": T, "s": dt, "complex_elem_updates_per_s": eu / dt}
print(json.dumps(res, indent=1))
