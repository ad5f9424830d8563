"""One config-2-shaped run (Haar n = 1e6, T = 100, tanh mix) for ncu captures;
DTYPE=f64|f32 (default f64)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
dtype = os.environ.get("DTYPE", "f64")
tdt = torch.float64 if dtype == "f64" else torch.float32
n = 1_000_000
op = lazymat.HaarOperator(n, seed=1, dtype=dtype, capacity=100)
x1 = torch.randn(n, dtype=tdt, device="cuda"); x1 /= x1.norm()
op.run(x1, 100, update="tanh_mix", sides="right")
torch.cuda.synchronize()
