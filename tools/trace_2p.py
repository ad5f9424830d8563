"""HD_TRACE=2 breakdown of the two-pass stage k_small_2p (config-2 shape)."""
import os, sys
os.environ["HD_TRACE"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
T = int(sys.argv[2]) if len(sys.argv) > 2 else 100
op = lazymat.HaarOperator(n, seed=1, capacity=T)
x = torch.randn(n, dtype=torch.float64, device="cuda")
x /= x.norm()
for _ in range(2):
    op.reset()
    op.run(x, T, update="tanh_mix", sides="right")
