import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2101_07464_b200 import lazymat as lm
n, T, seed = 1_000_000, 100, 12
x1 = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
x1 /= x1.norm(); x1 = x1.float().double()
a = lm.HaarOperator(n, seed=seed, capacity=T); b = lm.HaarOperator(n, seed=seed, dtype="f32", capacity=T)
ya = a.run(x1, T, update="tanh_mix", sides="right", keep_trajectory=True)
yb = b.run(x1.float(), T, update="tanh_mix", sides="right", keep_trajectory=True)
errs = [float((yb[t].double() - ya[t]).norm() / ya[t].norm()) for t in range(T + 1)]
print("max", max(errs), "at", errs.index(max(errs)), "last", errs[-1])
