import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2101_07464_b200 import lazymat
n = 1_000_000
op = lazymat.HaarOperator(n, seed=1, dtype="f32", capacity=100)
x1 = torch.randn(n, dtype=torch.float32, device="cuda"); x1 /= x1.norm()
op.run(x1, 100, update="tanh_mix", sides="right")
torch.cuda.synchronize()
