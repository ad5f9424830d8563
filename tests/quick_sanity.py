"""Fast GPU sanity check used while iterating (not collected by pytest)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as orc
from paper_2101_07464_b200 import lazymat

for n in (10, 1000, 70001):
    T = min(n, 12)
    ref = orc.Operator("haar", n=n, seed=3)
    op = lazymat.HaarOperator(n, seed=3, draws="injected", capacity=4)
    op.push_draws(orc.draws_for(3, [n] * T))
    aux = orc.RandomSource(4)
    worst = 0
    for t in range(T):
        x = aux.normal_vector(n)
        s = "left" if t % 3 == 0 else "right"
        worst = max(worst, np.linalg.norm(op.probe(x, s) - ref.probe(x, s)) / np.linalg.norm(x))
    print("haar", n, worst, flush=True)
m, n = 300, 257
ref = orc.Operator("ginibre", m=m, n=n, sigma=1.3, seed=5)
op = lazymat.GinibreOperator(m, n, sigma=1.3, seed=5, draws="injected", capacity=4)
sides = ["right", "left", "right", "right", "left", "left", "right"]
op.push_draws(orc.draws_for(5, [m if s == "right" else n for s in sides]))
aux = orc.RandomSource(6)
worst = 0
for s in sides:
    x = aux.normal_vector(n if s == "right" else m)
    worst = max(worst, np.linalg.norm(op.probe(x, s) - ref.probe(x, s)) / np.linalg.norm(x))
print("ginibre", worst, flush=True)
