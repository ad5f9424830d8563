"""BASELINE config 1 on the GPU: Ginibre m = n = 4096, sigma = 1/sqrt(n), T = 50
alternating probes, x_{t+1} = y/||y|| (device-resident run, graph replay);
median of 20 runs after warm-up, CUDA events."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat

n, T = 4096, 50
op = lazymat.GinibreOperator(n, n, n ** -0.5, 1, capacity=T)
x1 = torch.randn(n, dtype=torch.float64, device="cuda")
out = torch.empty(n, dtype=torch.float64, device="cuda")
times = []
for i in range(25):
    op.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.run_async(x1, T, out, update="normalize", sides="alternate", use_graph=True)
    op.wait()
    e1.record()
    torch.cuda.synchronize()
    if i >= 5:
        times.append(e0.elapsed_time(e1))
times.sort()
ms = times[len(times) // 2]
print(json.dumps({"workload": "config1_ginibre_4096_T50", "ms_per_run_median": ms,
                  "elem_updates_per_s": n * T * (T + 1) / 2 / (ms * 1e-3)}))
