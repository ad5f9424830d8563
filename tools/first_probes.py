"""A few probes of a fresh Haar operator at n = 1e6 (config 2 shape): the
fixed per-launch cost of the streaming kernels, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
n = int(os.environ.get("FP_N", 1_000_000))
op = lazymat.HaarOperator(n, seed=3, capacity=8)
x = torch.randn(n, dtype=torch.float64, device="cuda")
for t in range(int(os.environ.get("FP_T", 3))):
    x = op.probe(x, "right")
torch.cuda.synchronize()
print("ok")
