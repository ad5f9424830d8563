"""HD_TRACE=1 breakdown of the single-CTA stage (probe by probe, n = 1e6)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2101_07464_b200 import lazymat
n, T = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000, 60
op = lazymat.HaarOperator(n, seed=1, capacity=T)
x = torch.randn(n, dtype=torch.float64, device="cuda")
for t in range(T):
    x = op.probe(x / x.norm(), "right")
del op
