"""Attainable HBM bandwidth on this box for read-dominated streams
(torch reductions / copies over >> L2 buffers), timed with CUDA events."""
import json
import torch

def bench(fn, bytes_moved, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return bytes_moved / (best / 1e3) / 1e9

n = 100_000_000  # 800 MB fp64
x = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
m = x.view(100, -1)
v = torch.randn(m.shape[1], dtype=torch.float64, device="cuda")
res = {
    "sum_read_GBps": bench(lambda: x.sum(), 8 * n),
    "copy_rw_GBps": bench(lambda: y.copy_(x), 16 * n),
    "gemv_T_read_GBps": bench(lambda: m @ v, 8 * n),
    "gemv_N_read_GBps": bench(lambda: m.t() @ torch.ones(100, dtype=torch.float64, device="cuda"), 8 * n),
}
print(json.dumps(res))
